"""spconv-b200: the hot path of Hackel et al., arXiv 1801.10585, on B200 (sm_100a).

Sparse direct convolution with attention (Alg. 1), its sparsity-preserving backward (Alg. 2,
Eqs. (3)/(4)), sparse ReLU and sparse max-pooling, behind the C-ABI of include/spconv.h.
This package is the thin Python binding (argument marshalling only) plus the data-parallel
helper; all arithmetic runs in libspconv.so. It never imports `oracle/` and has no CPU
fallback: without the built library every op raises.
"""
from ._lib import SpconvError, load as _load_lib  # noqa: F401
from .ops import (  # noqa: F401
    SparseMap,
    SparseFilter,
    FwdPlan,
    BwdPlan,
    load,
    version,
    sparse_conv_fwd,
    sparse_conv_bwd,
    sparse_conv_bwd_input,
    sparse_conv_bwd_weight,
    round_f64,
    attention_topk,
    sparse_relu,
    sparse_maxpool,
    sparse_scatter_grad,
    select_variant,
    DensityReg,
    adagrad_step,
    filter_prune,
    sparse_to_dense,
    sparse_to_dense_bwd,
    encode_keys,
    decode_keys,
    memory_estimate,
    keys_narrow,
    keys_widen,
    kernel_launches,
    profile_enable,
    profile_reset,
    profile_read,
)
from . import dp  # noqa: F401
from . import spatial  # noqa: F401

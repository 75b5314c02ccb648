"""ORACLE — test infrastructure only (see oracle.c header).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import this package.
The product package `paper_1801_10585_b200` never imports it.
"""
from .oracle import (  # noqa: F401
    build,
    conv_fwd,
    conv_bwd,
    conv_bwd64,
    topk,
    relu,
    maxpool,
    scatter_grad,
    decode_key,
    encode_key,
    get_update_id,
    density_bias,
    adagrad_step,
    prune,
    to_dense,
    memory_estimate,
    ATTN_NONE,
    ATTN_MAGNITUDE,
    ATTN_RAW,
)

"""ctypes declaration of libspconv.so (include/spconv.h). Argument marshalling only."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libspconv.so")

MAX_NDIM = 4

STATUS = {
    0: "SPC_OK", 1: "SPC_ERR_INVALID_ARG", 2: "SPC_ERR_SHAPE", 3: "SPC_ERR_CAPACITY",
    4: "SPC_ERR_WORKSPACE", 5: "SPC_ERR_UNSORTED", 6: "SPC_ERR_UNSUPPORTED", 7: "SPC_ERR_CUDA",
}

ATTN = {"none": 0, "magnitude": 1, "raw": 2}
VARIANT = {"auto": 0, "scatter": 1, "gemm": 2}

# every symbol include/spconv.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "spc_version", "spc_status_string",
    "spc_conv_fwd_query", "sparse_conv_fwd",
    "spc_conv_fwd_query_ex", "sparse_conv_fwd_ex", "spc_conv_fwd_variant",
    "spc_conv_bwd_query", "sparse_conv_bwd", "sparse_conv_bwd_input", "sparse_conv_bwd_weight",
    "sparse_conv_bwd_f64", "spc_round_f64",
    "spc_topk_query", "attention_topk",
    "spc_relu_query", "sparse_relu",
    "spc_maxpool_query", "sparse_maxpool",
    "sparse_scatter_grad",
    "sparse_scatter_grad_sorted",
    "sparse_to_dense", "sparse_to_dense_bwd",
    "sparse_adagrad_step", "spc_prune_query", "sparse_filter_prune",
    "spc_conv_fwd_query_pass", "sparse_conv_fwd_pass",
    "spc_memory_estimate", "sparse_keys_narrow", "sparse_keys_widen",
    "spc_encode_keys", "spc_decode_keys",
    "spc_slab_gather_query", "spc_slab_gather", "spc_topk_digit_hist", "spc_topk_digit_pick",
    "spc_topk_keep_query", "spc_topk_keep_ge", "spc_index_add",
    "spc_kernel_launches", "spc_profile_enable", "spc_profile_reset", "spc_profile_read",
]


class MapT(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("batch", C.c_int64), ("channels", C.c_int64),
                ("dims", C.c_int64 * MAX_NDIM), ("nnz", C.c_int64), ("nnz_dev", C.c_void_p),
                ("keys", C.c_void_p), ("values", C.c_void_p), ("key_bits", C.c_int32)]


class MapOutT(C.Structure):
    _fields_ = [("capacity", C.c_int64), ("keys", C.c_void_p), ("values", C.c_void_p), ("nnz_dev", C.c_void_p),
                ("key_bits", C.c_int32)]


class FilterT(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("c_in", C.c_int64), ("c_out", C.c_int64),
                ("ksize", C.c_int64 * MAX_NDIM), ("nnz", C.c_int64), ("keys", C.c_void_p), ("values", C.c_void_p)]


class DensityRegT(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("rho_up", C.c_double), ("o", C.c_double), ("b1", C.c_double),
                ("b2", C.c_double)]


class SlabSrcT(C.Structure):
    _fields_ = [("keys", C.c_void_p), ("values", C.c_void_p), ("nnz_dev", C.c_void_p), ("n", C.c_int64),
                ("planes", C.c_int64), ("lo", C.c_int64), ("hi", C.c_int64), ("shift", C.c_int64)]


class SpconvError(RuntimeError):
    def __init__(self, fn: str, code: int):
        super().__init__(f"{fn} returned {STATUS.get(code, code)}")
        self.code = code


_lib = None


def load(path: str = LIB_PATH):
    """Load libspconv.so. Fails loudly when the library is missing: there is no fallback.
    SPC_LIB=<path> selects another build of the same library (e.g. libspconv_debug.so)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SPC_LIB", path)
    if not os.path.exists(path):
        raise ImportError(f"libspconv.so not found at {path}; run `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no CPU fallback)")
    lib = C.CDLL(path)
    P = C.c_void_p
    I64 = C.c_int64
    pM, pO, pF = C.POINTER(MapT), C.POINTER(MapOutT), C.POINTER(FilterT)
    sz = C.POINTER(C.c_size_t)
    pi64 = C.POINTER(C.c_int64)
    sig = {
        "spc_version": ([], C.c_char_p),
        "spc_status_string": ([C.c_int], C.c_char_p),
        "spc_conv_fwd_query": ([pM, pF, C.c_int, I64, pi64, sz], C.c_int),
        "sparse_conv_fwd": ([pM, pF, P, C.c_int, I64, pO, P, C.c_size_t, P], C.c_int),
        "spc_conv_fwd_query_ex": ([pM, pF, C.c_int, I64, C.c_int, pi64, sz], C.c_int),
        "sparse_conv_fwd_ex": ([pM, pF, P, C.c_int, I64, C.c_int, pO, P, C.c_size_t, P], C.c_int),
        "spc_conv_fwd_variant": ([pM, pF, C.c_int, I64, C.c_int], C.c_int),
        "spc_conv_bwd_query": ([pM, pF, pM, sz], C.c_int),
        "sparse_conv_bwd": ([pM, pF, pM, P, P, P, P, P, C.c_size_t, P], C.c_int),
        "sparse_conv_bwd_input": ([pM, pF, pM, P, P, P, C.c_size_t, P], C.c_int),
        "sparse_conv_bwd_weight": ([pM, pF, pM, P, P, P, P, C.c_size_t, P], C.c_int),
        "sparse_conv_bwd_f64": ([pM, pF, pM, P, P, P, P, P, C.c_size_t, P], C.c_int),
        "spc_round_f64": ([P, P, I64, P], C.c_int),
        "spc_topk_query": ([pM, C.c_int, I64, pi64, sz], C.c_int),
        "attention_topk": ([pM, C.c_int, I64, pO, P, P, C.c_size_t, P], C.c_int),
        "spc_relu_query": ([pM, pi64, sz], C.c_int),
        "sparse_relu": ([pM, pO, P, P, C.c_size_t, P], C.c_int),
        "spc_maxpool_query": ([pM, P, pi64, sz], C.c_int),
        "sparse_maxpool": ([pM, P, pO, P, P, C.c_size_t, P], C.c_int),
        "sparse_scatter_grad": ([P, P, I64, P, P, I64, P], C.c_int),
        "sparse_scatter_grad_sorted": ([P, P, I64, P, P, I64, P], C.c_int),
        "sparse_adagrad_step": ([P, P, P, I64, P, C.c_double, C.POINTER(DensityRegT), C.c_double, C.c_double, P],
                                C.c_int),
        "spc_prune_query": ([I64, sz], C.c_int),
        "sparse_to_dense": ([pM, P, P], C.c_int),
        "sparse_to_dense_bwd": ([pM, P, P, P], C.c_int),
        "sparse_filter_prune": ([P, P, P, P, I64, C.c_double, P, P, P, P, P, P, C.c_size_t, P], C.c_int),
        "spc_conv_fwd_query_pass": ([pM, pF, C.c_int, I64, I64, pi64, sz], C.c_int),
        "sparse_conv_fwd_pass": ([pM, pF, P, C.c_int, I64, I64, pO, P, C.c_size_t, P], C.c_int),
        "spc_memory_estimate": ([C.c_int32, I64, I64, I64, C.c_double, C.c_int32, C.POINTER(C.c_double),
                                 C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
        "sparse_keys_narrow": ([pM, P, P], C.c_int),
        "sparse_keys_widen": ([P, P, I64, P, P], C.c_int),
        "spc_encode_keys": ([C.c_int32, I64, I64, P, P, I64, P, P, P], C.c_int),
        "spc_decode_keys": ([C.c_int32, I64, I64, P, P, I64, P, P, P], C.c_int),
        "spc_slab_gather_query": ([I64, C.c_int32, sz], C.c_int),
        "spc_slab_gather": ([C.POINTER(SlabSrcT), C.c_int32, I64, I64, I64, pO, P, P, C.c_size_t, P], C.c_int),
        "spc_topk_digit_hist": ([pM, C.c_int, I64, P, P, C.c_int32, P, P], C.c_int),
        "spc_topk_digit_pick": ([I64, P, C.c_int32, P, P, P], C.c_int),
        "spc_topk_keep_query": ([pM, sz], C.c_int),
        "spc_topk_keep_ge": ([pM, C.c_int, I64, P, pO, P, P, C.c_size_t, P], C.c_int),
        "spc_index_add": ([P, P, I64, P, P, P], C.c_int),
        "spc_kernel_launches": ([], C.c_int64),
        "spc_profile_enable": ([C.c_int], C.c_int),
        "spc_profile_reset": ([], C.c_int),
        "spc_profile_read": ([C.c_char_p, C.c_size_t, P, P, C.c_int], C.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def check(fn: str, code: int):
    if code != 0:
        raise SpconvError(fn, code)

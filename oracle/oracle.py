"""ctypes binding of the C oracle (oracle.c). TEST INFRASTRUCTURE ONLY.

Argument marshalling only; every step of the arithmetic is in oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ATTN_NONE, ATTN_MAGNITUDE, ATTN_RAW = 0, 1, 2

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2, no fast-math: IEEE semantics are part of the oracle)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        I64 = C.c_int64
        _lib.ora_conv_fwd.argtypes = [C.c_int, P, I64, I64, I64, P, I64, P, P, I64, P, P, P, C.c_int, I64,
                                      I64, P, P, P, P, P]
        _lib.ora_conv_bwd.argtypes = [C.c_int, P, I64, I64, I64, P, I64, P, P, I64, P, P, I64, P, P,
                                      P, P, P, P, P, P]
        _lib.ora_conv_bwd64.argtypes = [C.c_int, P, I64, I64, I64, P, I64, P, P, I64, P, P, I64, P, P,
                                        P, P, P, P, P, P, P, P]
        _lib.ora_topk.argtypes = [C.c_int, P, I64, I64, I64, P, P, C.c_int, I64, I64, P, P, P, P]
        _lib.ora_relu.argtypes = [I64, P, P, P, P, P, P]
        _lib.ora_maxpool.argtypes = [C.c_int, P, I64, I64, P, I64, P, P, I64, P, P, P, P]
        _lib.ora_scatter_grad.argtypes = [I64, P, P, I64, P]
        _lib.ora_decode_key.argtypes = [C.c_uint64, C.c_int, P, I64, I64, P]
        _lib.ora_encode_key.argtypes = [C.c_int, P, I64, P]
        _lib.ora_encode_key.restype = C.c_uint64
        _lib.ora_get_update_id.argtypes = [C.c_int, P, P, P, P, P]
        _lib.ora_density_bias.argtypes = [C.c_double] * 5
        _lib.ora_density_bias.restype = C.c_double
        _lib.ora_adagrad_step.argtypes = [I64, P, P, P, C.c_double, C.c_double, C.c_double, C.c_double]
        _lib.ora_adagrad_step.restype = C.c_int
        _lib.ora_prune.argtypes = [I64, P, P, P, P, C.c_double, P, P, P, P]
        _lib.ora_prune.restype = C.c_int64
        _lib.ora_to_dense.argtypes = [C.c_int, P, I64, I64, I64, P, P, P]
        _lib.ora_to_dense.restype = C.c_int
        _lib.ora_memory_estimate.argtypes = [C.c_int, I64, I64, I64, C.c_double, C.c_int, P]
        _lib.ora_memory_estimate.restype = C.c_int
        for f in ("ora_conv_fwd", "ora_conv_bwd", "ora_conv_bwd64", "ora_topk", "ora_relu", "ora_maxpool",
                  "ora_scatter_grad", "ora_decode_key", "ora_get_update_id"):
            getattr(_lib, f).restype = C.c_int
    return _lib


class OracleError(RuntimeError):
    pass


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _i64(seq) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(seq, dtype=np.int64))


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _check(rc: int, what: str):
    if rc != 0:
        raise OracleError(f"{what} failed with code {rc}")


def decode_key(key: int, dims: Sequence[int], batch: int, channels: int):
    out = np.zeros(2 + len(dims), np.int64)
    _check(_load().ora_decode_key(int(key), len(dims), _p(_i64(dims)), batch, channels, _p(out)), "decode_key")
    return tuple(int(v) for v in out)


def encode_key(idx: Sequence[int], dims: Sequence[int], channels: int) -> int:
    return int(_load().ora_encode_key(len(dims), _p(_i64(dims)), channels, _p(_i64(idx))))


def get_update_id(id_, fid, dims, ksize):
    uid = np.zeros(len(dims), np.int64)
    ok = _load().ora_get_update_id(len(dims), _p(_i64(dims)), _p(_i64(ksize)), _p(_i64(id_)), _p(_i64(fid)), _p(uid))
    return tuple(int(v) for v in uid) if ok else None


def conv_fwd(x, w, bias, attn: int = ATTN_NONE, k: int = 0, with_abs: bool = False):
    """Alg. 1. x: synth.COO, w: synth.Filter, bias: float32[c_out] or None.
    Returns (keys, values, abs_or_None, macs)."""
    dims = _i64(x.dims)
    ks = _i64(w.ksize)
    V = int(np.prod(x.dims))
    per = min(k, V) if attn else V
    cap = max(1, x.batch * w.c_out * per)
    yk = np.zeros(cap, np.uint64)
    yv = np.zeros(cap, np.float32)
    ya = np.zeros(cap, np.float64) if with_abs else None
    ny = np.zeros(1, np.int64)
    macs = np.zeros(1, np.int64)
    xk, xv, wk, wv = _u64(x.keys), _f32(x.values), _u64(w.keys), _f32(w.values)
    b = None if bias is None else _f32(bias)
    rc = _load().ora_conv_fwd(x.ndim, _p(dims), x.batch, w.c_in, w.c_out, _p(ks),
                              x.nnz, _p(xk), _p(xv), w.nnz, _p(wk), _p(wv), _p(b), int(attn), int(k),
                              cap, _p(yk), _p(yv), _p(ya), _p(ny), _p(macs))
    _check(rc, "ora_conv_fwd")
    n = int(ny[0])
    return yk[:n].copy(), yv[:n].copy(), (ya[:n].copy() if with_abs else None), int(macs[0])


def conv_bwd(x, w, y_keys, dy, with_abs: bool = False, return_pairs: bool = False):
    """Alg. 2. Returns (dx, dw, dbias, dx_abs, dw_abs) [+ number of (input, weight) pairs whose
    target is a kept output, when return_pairs]."""
    dims = _i64(x.dims)
    ks = _i64(w.ksize)
    xk, xv, wk, wv = _u64(x.keys), _f32(x.values), _u64(w.keys), _f32(w.values)
    yk, g = _u64(y_keys), _f32(dy)
    dx = np.zeros(max(1, x.nnz), np.float32)
    dw = np.zeros(max(1, w.nnz), np.float32)
    db = np.zeros(w.c_out, np.float32)
    dxa = np.zeros(max(1, x.nnz), np.float64) if with_abs else None
    dwa = np.zeros(max(1, w.nnz), np.float64) if with_abs else None
    pairs = np.zeros(1, np.int64)
    rc = _load().ora_conv_bwd(x.ndim, _p(dims), x.batch, w.c_in, w.c_out, _p(ks),
                              x.nnz, _p(xk), _p(xv), w.nnz, _p(wk), _p(wv), yk.shape[0], _p(yk), _p(g),
                              _p(dx), _p(dw), _p(db), _p(dxa), _p(dwa), _p(pairs))
    _check(rc, "ora_conv_bwd")
    out = (dx[:x.nnz], dw[:w.nnz], db,
           dxa[:x.nnz] if with_abs else None, dwa[:w.nnz] if with_abs else None)
    return out + (int(pairs[0]),) if return_pairs else out


def conv_bwd64(x, w, y_keys, dy, with_abs: bool = False):
    """Alg. 2 with the fp64 sums of dw / dbias before their rounding (per-shard partials for the
    data-parallel tests). Returns (dx, dw64, db64, dx_abs, dw_abs)."""
    dims = _i64(x.dims)
    ks = _i64(w.ksize)
    xk, xv, wk, wv = _u64(x.keys), _f32(x.values), _u64(w.keys), _f32(w.values)
    yk, g = _u64(y_keys), _f32(dy)
    dx = np.zeros(max(1, x.nnz), np.float32)
    dw = np.zeros(max(1, w.nnz), np.float32)
    db = np.zeros(w.c_out, np.float32)
    dw64 = np.zeros(max(1, w.nnz), np.float64)
    db64 = np.zeros(w.c_out, np.float64)
    dxa = np.zeros(max(1, x.nnz), np.float64) if with_abs else None
    dwa = np.zeros(max(1, w.nnz), np.float64) if with_abs else None
    pairs = np.zeros(1, np.int64)
    rc = _load().ora_conv_bwd64(x.ndim, _p(dims), x.batch, w.c_in, w.c_out, _p(ks),
                                x.nnz, _p(xk), _p(xv), w.nnz, _p(wk), _p(wv), yk.shape[0], _p(yk), _p(g),
                                _p(dx), _p(dw), _p(db), _p(dxa), _p(dwa), _p(pairs), _p(dw64), _p(db64))
    _check(rc, "ora_conv_bwd64")
    return (dx[:x.nnz], dw64[:w.nnz], db64,
            dxa[:x.nnz] if with_abs else None, dwa[:w.nnz] if with_abs else None)


def topk(x, attn: int, k: int):
    """Standalone attention (k-selection per (b, c) segment). Returns (keys, values, src)."""
    dims = _i64(x.dims)
    V = int(np.prod(x.dims))
    cap = max(1, min(x.nnz, x.batch * x.channels * min(k, V)))
    yk = np.zeros(cap, np.uint64)
    yv = np.zeros(cap, np.float32)
    src = np.zeros(cap, np.int64)
    ny = np.zeros(1, np.int64)
    xk, xv = _u64(x.keys), _f32(x.values)
    rc = _load().ora_topk(x.ndim, _p(dims), x.batch, x.channels, x.nnz, _p(xk), _p(xv), int(attn), int(k),
                          cap, _p(yk), _p(yv), _p(src), _p(ny))
    _check(rc, "ora_topk")
    n = int(ny[0])
    return yk[:n].copy(), yv[:n].copy(), src[:n].copy()


def relu(x):
    cap = max(1, x.nnz)
    yk = np.zeros(cap, np.uint64)
    yv = np.zeros(cap, np.float32)
    src = np.zeros(cap, np.int64)
    ny = np.zeros(1, np.int64)
    xk, xv = _u64(x.keys), _f32(x.values)
    _check(_load().ora_relu(x.nnz, _p(xk), _p(xv), _p(yk), _p(yv), _p(src), _p(ny)), "ora_relu")
    n = int(ny[0])
    return yk[:n].copy(), yv[:n].copy(), src[:n].copy()


def maxpool(x, stride: Sequence[int]):
    """Returns (keys, values, argmax) of the pooled map (dims ceil(d/s))."""
    dims = _i64(x.dims)
    st = _i64(stride)
    cap = max(1, x.nnz)
    yk = np.zeros(cap, np.uint64)
    yv = np.zeros(cap, np.float32)
    am = np.zeros(cap, np.int64)
    ny = np.zeros(1, np.int64)
    xk, xv = _u64(x.keys), _f32(x.values)
    rc = _load().ora_maxpool(x.ndim, _p(dims), x.batch, x.channels, _p(st), x.nnz, _p(xk), _p(xv),
                             cap, _p(yk), _p(yv), _p(am), _p(ny))
    _check(rc, "ora_maxpool")
    n = int(ny[0])
    return yk[:n].copy(), yv[:n].copy(), am[:n].copy()


def scatter_grad(src, dy, nx: int):
    s = _i64(src)
    g = _f32(dy)
    dx = np.zeros(max(1, nx), np.float32)
    _check(_load().ora_scatter_grad(s.shape[0], _p(s), _p(g), nx, _p(dx)), "ora_scatter_grad")
    return dx[:nx]


# ------------------------------------------------------------------ training-loop steps (f1)
def density_bias(rho: float, rho_up: float, o: float = 0.1, b1: float = 0.1, b2: float = 0.1) -> float:
    """Eq. (6)."""
    return float(_load().ora_density_bias(rho, rho_up, o, b1, b2))


def adagrad_step(w, dw, acc, b: float, lam: float, lr: float, eps: float):
    """One Adagrad step with the density regulariser (§3.5, §4); returns new (w, acc) as fp32."""
    w = np.ascontiguousarray(w, np.float32).copy()
    acc = np.ascontiguousarray(acc, np.float32).copy()
    dw = np.ascontiguousarray(dw, np.float32)
    rc = _load().ora_adagrad_step(w.size, w.ctypes.data, dw.ctypes.data, acc.ctypes.data, b, lam, lr, eps)
    if rc != 0:
        raise OracleError(f"ora_adagrad_step rc={rc}")
    return w, acc


def prune(keys, w, acc, warn, eps: float = 0.01):
    """One-warning-shot pruning (§3.6); returns compacted (keys, w, acc, warn)."""
    keys = np.ascontiguousarray(keys, np.uint64)
    w = np.ascontiguousarray(w, np.float32)
    acc = np.ascontiguousarray(acc, np.float32)
    warn = np.ascontiguousarray(warn, np.uint8)
    n = keys.size
    ok, ow, oa, owr = (np.zeros(max(n, 1), np.uint64), np.zeros(max(n, 1), np.float32),
                       np.zeros(max(n, 1), np.float32), np.zeros(max(n, 1), np.uint8))
    m = _load().ora_prune(n, keys.ctypes.data, w.ctypes.data, acc.ctypes.data, warn.ctypes.data, eps,
                          ok.ctypes.data, ow.ctypes.data, oa.ctypes.data, owr.ctypes.data)
    if m < 0:
        raise OracleError("ora_prune failed")
    return ok[:m], ow[:m], oa[:m], owr[:m]


def to_dense(x):
    """sparseToDense() (Table 2): dense [batch, channels, *dims] float32 array."""
    dims = np.asarray(x.dims, np.int64)
    out = np.zeros((x.batch, x.channels) + tuple(x.dims), np.float32)
    keys = np.ascontiguousarray(x.keys, np.uint64)
    vals = np.ascontiguousarray(x.values, np.float32)
    rc = _load().ora_to_dense(len(x.dims), dims.ctypes.data, x.batch, x.channels, keys.size, keys.ctypes.data,
                              vals.ctypes.data, out.ctypes.data)
    if rc != 0:
        raise OracleError(f"ora_to_dense rc={rc}")
    return out


# ------------------------------------------------------------------ memory model (f2)
def memory_estimate(k: int, r: int, b: int, c: int, rho_up: float, index_bits: int = 64):
    """Table 1 / Fig. 7: {"dense", "sparse", "temp"} bytes, or None for
    32-bit indices past 2^32 cells (the paper's overflow caveat)."""
    out = np.zeros(3, np.float64)
    rc = _load().ora_memory_estimate(int(k), int(r), int(b), int(c), float(rho_up), int(index_bits), _p(out))
    if rc < 0:
        return None
    return {"dense": float(out[0]), "sparse": float(out[1]), "temp": float(out[2])}

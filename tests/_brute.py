"""Brute-force references that pin the oracle (tests only).

These are independent of oracle.c: dense fp64 cross-correlation via torch's CPU convolution
(a library routine), a plain numpy shift-and-add definition for any rank, dense autograd, and
Python full sorts. Nothing here is shared with the CUDA path.
"""
from __future__ import annotations

import itertools

import numpy as np
import torch
import torch.nn.functional as F


def coo_to_dense(x):
    """[B, C, *dims] float64 values and bool presence."""
    B, Cc, dims = x.batch, x.channels, tuple(x.dims)
    V = int(np.prod(dims))
    val = np.zeros(B * Cc * V, np.float64)
    pres = np.zeros(B * Cc * V, bool)
    k = x.keys.astype(np.int64)
    val[k] = x.values.astype(np.float64)
    pres[k] = True
    return val.reshape((B, Cc) + dims), pres.reshape((B, Cc) + dims)


def filter_to_dense(w):
    """[c_out, c_in, *ksize] float64 values and bool presence."""
    K = int(np.prod(w.ksize))
    val = np.zeros(w.c_out * w.c_in * K, np.float64)
    pres = np.zeros(w.c_out * w.c_in * K, bool)
    k = w.keys.astype(np.int64)
    val[k] = w.values.astype(np.float64)
    pres[k] = True
    return val.reshape((w.c_out, w.c_in) + tuple(w.ksize)), pres.reshape((w.c_out, w.c_in) + tuple(w.ksize))


def torch_xcorr(X, W):
    """Dense SAME cross-correlation in float64 via torch.nn.functional.conv{1,2,3}d."""
    nd = X.ndim - 2
    conv = {1: F.conv1d, 2: F.conv2d, 3: F.conv3d}[nd]
    pad = tuple(int(k) // 2 for k in W.shape[2:])
    return conv(torch.from_numpy(X), torch.from_numpy(W), padding=pad).numpy()


def shift_xcorr(X, W):
    """Dense SAME cross-correlation for any rank from its definition:
    out[b, oc, p] = sum_{ic, delta} W[oc, ic, delta] * X[b, ic, p + delta - c] (zero outside)."""
    B, Cin = X.shape[:2]
    dims = X.shape[2:]
    Cout = W.shape[0]
    ks = W.shape[2:]
    out = np.zeros((B, Cout) + dims, np.float64)
    pads = [(0, 0), (0, 0)] + [(k // 2, k // 2) for k in ks]
    Xp = np.pad(X, pads)
    for delta in itertools.product(*[range(k) for k in ks]):
        sl = tuple(slice(d, d + n) for d, n in zip(delta, dims))
        xs = Xp[(slice(None), slice(None)) + sl]  # X[p + delta - c]
        wd = W[(slice(None), slice(None)) + tuple(delta)]  # [Cout, Cin]
        out += np.einsum("oi,bi...->bo...", wd, xs)
    return out


def dense_to_sorted(Y, mask):
    """keys (row-major over [B, C, *dims]) and values of the masked entries."""
    flat = mask.reshape(-1)
    keys = np.nonzero(flat)[0].astype(np.uint64)
    return keys, Y.reshape(-1)[flat]


def brute_topk(keys, values, V, k, attn):
    """Per segment (key // V) keep the first k under (score desc, key asc) via a full Python sort."""
    segs = {}
    for kk, v in zip(keys.tolist(), values.tolist()):
        segs.setdefault(kk // V, []).append((kk, v))
    kept = []
    for s in sorted(segs):
        ent = segs[s]
        score = (lambda v: abs(v)) if attn == "magnitude" else (lambda v: v)
        ent = sorted(ent, key=lambda e: (-score(e[1]), e[0]))[:k]
        kept.extend(sorted(ent))
    return np.array([e[0] for e in kept], np.uint64), np.array([e[1] for e in kept], np.float32)


def masked_conv_grads(x, w, bias, y_keys, dy):
    """fp64 autograd of L = sum_{kept p} dy_p * (xcorr(X, W) + bias)_p, X/W dense with zeros at
    non-stored coordinates; returns dense dX, dW, dbias (to be read at the stored coordinates)."""
    Xd, _ = coo_to_dense(x)
    Wd, _ = filter_to_dense(w)
    nd = Xd.ndim - 2
    conv = {1: F.conv1d, 2: F.conv2d, 3: F.conv3d}[nd]
    X = torch.from_numpy(Xd).requires_grad_(True)
    W = torch.from_numpy(Wd).requires_grad_(True)
    b = torch.from_numpy(np.asarray(bias, np.float64)).requires_grad_(True)
    pad = tuple(int(k) // 2 for k in w.ksize)
    Y = conv(X, W, padding=pad) + b.view((1, -1) + (1,) * nd)
    G = torch.zeros(Y.numel(), dtype=torch.float64)
    G[torch.from_numpy(y_keys.astype(np.int64))] = torch.from_numpy(dy.astype(np.float64))
    L = (Y.reshape(-1) * G).sum()
    L.backward()
    return X.grad.numpy(), W.grad.numpy(), b.grad.numpy()

"""Parity of the CUDA path (through the C-ABI) with the CPU oracle on identical seeded inputs.

Bar: keys, masks, argmax and src indices bit-exact; with dyadic
inputs every value and gradient bit-exact too (all fp32 sums exact in any order); with
continuous inputs |gpu - ora| <= 1e-5 |ora| + 1e-6 sum|terms| and attention sets equal up to
near-threshold swaps.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle as ora
from synth import (COO, Filter, uniform_map, mnist_like, surface_occupancy, sparse_filter, bias_vector, grad_values,
                   select_samples, SEED_BASE)
from tests._compare import assert_values_close, assert_topk_sets_match

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ATTN_ORA = {"none": ora.ATTN_NONE, "magnitude": ora.ATTN_MAGNITUDE, "raw": ora.ATTN_RAW}


def dev_map(spc, x: COO):
    return spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)


def dev_filter(spc, w: Filter):
    return spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)


def host(t):
    return t.detach().cpu().numpy()


def host_keys(t):
    return host(t).view(np.uint64)


def run_fwd(spc, x, w, bias, attn, k, variant="scatter"):
    y = spc.sparse_conv_fwd(dev_map(spc, x), dev_filter(spc, w),
                            None if bias is None else torch.from_numpy(bias).cuda(), attn, k, variant=variant)
    yk, yv = y.trimmed()
    return host_keys(yk), host(yv), y


FWD_CASES = [
    # name, dims, batch, c_in, c_out, ksize, rho_d, rho_f
    ("1d", (37,), 3, 2, 3, (3,), 0.2, 0.7),
    ("2d_8x8", (8, 8), 2, 2, 3, (3, 3), 0.2, 0.5),
    ("2d_5x3k", (13, 17), 2, 3, 5, (5, 3), 0.1, 0.8),
    ("3d_small", (9, 7, 11), 2, 3, 4, (3, 3, 3), 0.08, 0.5),
    ("3d_tiles", (24, 20, 40), 2, 8, 8, (3, 3, 3), 0.03, 0.5),   # several tiles + ragged tail
    ("3d_k1", (6, 6, 6), 2, 4, 6, (1, 1, 1), 0.3, 1.0),
    ("3d_wide_oc", (10, 12, 14), 1, 2, 40, (3, 3, 3), 0.05, 0.3),  # several oc groups
    ("3d_long_z", (3, 3, 700), 2, 2, 3, (3, 3, 3), 0.05, 0.5),
    ("3d_dense", (12, 16, 64), 1, 3, 4, (3, 3, 3), 0.4, 0.5),     # > 32 inputs per warp item
    ("3d_z128", (5, 9, 128), 2, 3, 4, (3, 3, 3), 0.05, 0.5),      # Z a multiple of 128
]


@pytest.mark.parametrize("case", FWD_CASES, ids=lambda c: c[0])
@pytest.mark.parametrize("attn", ["none", "magnitude", "raw"])
def test_fwd_dyadic_bit_exact(cuda_lib, case, attn):
    spc = cuda_lib
    _, dims, B, ci, co, ks, rd, rf = case
    x = uniform_map(B, ci, dims, rd, 1000 + len(dims), values="dyadic")
    w = sparse_filter(ci, co, ks, rf, 1001, values="dyadic")
    bias = bias_vector(co, 1002, values="dyadic")
    V = int(np.prod(dims))
    k = max(1, V // 20)
    ok_, ov, _, _ = ora.conv_fwd(x, w, bias, attn=ATTN_ORA[attn], k=k)
    gk, gv, _ = run_fwd(spc, x, w, bias, attn, k)
    np.testing.assert_array_equal(gk, ok_)
    np.testing.assert_array_equal(gv, ov)


@pytest.mark.parametrize("case", FWD_CASES, ids=lambda c: c[0])
@pytest.mark.parametrize("attn", ["none", "magnitude", "raw"])
def test_fwd_continuous_tolerance(cuda_lib, case, attn):
    spc = cuda_lib
    _, dims, B, ci, co, ks, rd, rf = case
    x = uniform_map(B, ci, dims, rd, 2000 + len(dims))
    w = sparse_filter(ci, co, ks, rf, 2001)
    bias = bias_vector(co, 2002)
    V = int(np.prod(dims))
    k = max(1, V // 20)
    fk, fv, fa, _ = ora.conv_fwd(x, w, bias, with_abs=True)           # exact support + scales
    gk, gv, _ = run_fwd(spc, x, w, bias, attn, k)
    if attn == "none":
        np.testing.assert_array_equal(gk, fk)                           # structural support: exact
        assert_values_close(gv, fv, fa)
        return
    ok_, ov, _, _ = ora.conv_fwd(x, w, bias, attn=ATTN_ORA[attn], k=k)
    assert_topk_sets_match(gk, gv, ok_, ov, fk, fv, fa, V, k, attn)
    # values at common keys
    common, gi, oi = np.intersect1d(gk, ok_, return_indices=True)
    idx = np.searchsorted(fk, common)
    assert_values_close(gv[gi], ov[oi], fa[idx])


# ------------------------------------------------------------ rank 4 ("generic n-dimensional")
RANK4_CASES = [
    # name, dims, batch, c_in, c_out, ksize, rho_d, rho_f
    ("4d_small", (5, 6, 7, 9), 2, 3, 4, (3, 3, 3, 3), 0.05, 0.4),
    ("4d_k3133", (4, 5, 6, 8), 1, 2, 5, (3, 1, 3, 3), 0.1, 0.6),
    ("4d_k5w", (7, 4, 4, 12), 2, 2, 3, (5, 3, 1, 3), 0.08, 0.5),
    ("4d_sampled", (12, 16, 20, 32), 1, 2, 3, (3, 3, 3, 3), 0.02, 0.3),   # sampled threshold (>= 184 tiles)
]


@pytest.mark.parametrize("case", RANK4_CASES, ids=lambda c: c[0])
@pytest.mark.parametrize("attn", ["none", "magnitude", "raw"])
@pytest.mark.parametrize("values", ["dyadic", "continuous"])
def test_fwd_rank4(cuda_lib, case, attn, values):
    spc = cuda_lib
    _, dims, B, ci, co, ks, rd, rf = case
    x = uniform_map(B, ci, dims, rd, 4400, values=values)
    w = sparse_filter(ci, co, ks, rf, 4401, values=values)
    bias = bias_vector(co, 4402, values=values)
    V = int(np.prod(dims))
    k = max(1, V // 20)
    gk, gv, _ = run_fwd(spc, x, w, bias, attn, k, variant="auto")
    if values == "dyadic":
        ok_, ov, _, _ = ora.conv_fwd(x, w, bias, attn=ATTN_ORA[attn], k=k)
        np.testing.assert_array_equal(gk, ok_)
        np.testing.assert_array_equal(gv, ov)
        return
    fk, fv, fa, _ = ora.conv_fwd(x, w, bias, with_abs=True)
    if attn == "none":
        np.testing.assert_array_equal(gk, fk)
        assert_values_close(gv, fv, fa)
        return
    ok_, ov, _, _ = ora.conv_fwd(x, w, bias, attn=ATTN_ORA[attn], k=k)
    assert_topk_sets_match(gk, gv, ok_, ov, fk, fv, fa, V, k, attn)


@pytest.mark.parametrize("case", RANK4_CASES[:3], ids=lambda c: c[0])
@pytest.mark.parametrize("values", ["dyadic", "continuous"])
def test_bwd_rank4(cuda_lib, case, values):
    spc = cuda_lib
    _, dims, B, ci, co, ks, rd, rf = case
    x = uniform_map(B, ci, dims, rd, 4500, values=values)
    w = sparse_filter(ci, co, ks, rf, 4501, values=values)
    bias = bias_vector(co, 4502, values=values)
    V = int(np.prod(dims))
    yk, yv, _, _ = ora.conv_fwd(x, w, bias, attn=ora.ATTN_MAGNITUDE, k=max(1, V // 10))
    dy = grad_values(yk.shape[0], 4503, values=values)
    dx, dw, db, dxa, dwa = ora.conv_bwd(x, w, yk, dy, with_abs=True)
    Y = spc.SparseMap.from_arrays(yk, yv, B, co, dims)
    gdx, gdw, gdb = (host(t) for t in spc.sparse_conv_bwd(dev_map(spc, x), dev_filter(spc, w), Y,
                                                           torch.from_numpy(dy).cuda()))
    if values == "dyadic":
        np.testing.assert_array_equal(gdx, dx)
        np.testing.assert_array_equal(gdw, dw)
        np.testing.assert_array_equal(gdb, db)
    else:
        assert_values_close(gdx, dx, dxa, "dx")
        assert_values_close(gdw, dw, dwa, "dw")


@pytest.mark.parametrize("dims,stride", [((6, 8, 8, 10), (2, 2, 2, 2)), ((5, 7, 4, 9), (3, 1, 2, 4)),
                                         ((3, 2, 3, 9000), (1, 2, 1, 2)),    # PZ 4500 > 4096: the row form
                                         ((16, 18, 4, 6), (8, 9, 1, 2))])    # sw * sx = 72 > 64 planes: row form
def test_maxpool_relu_topk_rank4(cuda_lib, dims, stride):
    spc = cuda_lib
    x = uniform_map(2, 3, dims, 0.3, 4600, values="dyadic")
    ok_, ov, oarg = ora.maxpool(x, stride)
    y, arg = spc.sparse_maxpool(dev_map(spc, x), stride)
    yk, yv = y.trimmed()
    np.testing.assert_array_equal(host_keys(yk), ok_)
    np.testing.assert_array_equal(host(yv), ov)
    np.testing.assert_array_equal(host(arg[:yk.shape[0]]), oarg)
    rk, rv, rsrc = ora.relu(x)
    y, src = spc.sparse_relu(dev_map(spc, x))
    np.testing.assert_array_equal(host_keys(y.trimmed()[0]), rk)
    k = 17
    tk, tv, tsrc = ora.topk(x, ora.ATTN_MAGNITUDE, k)
    y, src = spc.attention_topk(dev_map(spc, x), "magnitude", k)
    yk, yv = y.trimmed()
    np.testing.assert_array_equal(host_keys(yk), tk)
    np.testing.assert_array_equal(host(yv), tv)


# ---------------------------------------------------------------- variant G (tcgen05, 3xTF32)
GEMM_CASES = FWD_CASES + [
    # C5-like: 32 -> 32 channels, dense filter, several densities (SURVEY §8 d, C5)
    ("c5_like_5pct", (10, 12, 32), 2, 32, 32, (3, 3, 3), 0.05, 1.0),
    ("c5_like_30pct", (6, 8, 32), 1, 32, 32, (3, 3, 3), 0.3, 1.0),
    ("c3_like_32_64", (8, 8, 24), 1, 32, 64, (3, 3, 3), 0.1, 0.6),
    ("ksplit_16ch", (9, 37, 20), 2, 16, 24, (3, 3, 3), 0.15, 0.7),      # Kp 16: two K parts; ragged bands
    ("kp24_noswizzle", (7, 9, 30), 1, 20, 8, (3, 3, 3), 0.2, 0.5),      # Kp 24: one part, plain slots
    ("long_z_densify_fallback", (2, 3, 4000), 1, 3, 4, (3, 3, 3), 0.05, 0.6),   # band > smem: scatter densify
]


@pytest.mark.parametrize("case", GEMM_CASES, ids=lambda c: c[0])
@pytest.mark.parametrize("attn", ["none", "magnitude"])
def test_fwd_gemm_dyadic_bit_exact(cuda_lib, case, attn):
    """Variant G must reproduce the oracle bit for bit on dyadic data (TF32 holds the 7-bit
    dyadic operands exactly, every partial sum is exact) -- same support, same selection."""
    spc = cuda_lib
    _, dims, B, ci, co, ks, rd, rf = case
    x = uniform_map(B, ci, dims, rd, 3000 + len(dims), values="dyadic")
    w = sparse_filter(ci, co, ks, rf, 3001, values="dyadic4" if ci >= 16 else "dyadic")
    bias = bias_vector(co, 3002, values="dyadic")
    V = int(np.prod(dims))
    k = max(1, V // 20)
    ok_, ov, _, _ = ora.conv_fwd(x, w, bias, attn=ATTN_ORA[attn], k=k)
    gk, gv, _ = run_fwd(spc, x, w, bias, attn, k, variant="gemm")
    np.testing.assert_array_equal(gk, ok_)
    np.testing.assert_array_equal(gv, ov)


@pytest.mark.parametrize("case", GEMM_CASES, ids=lambda c: c[0])
def test_fwd_gemm_continuous_tolerance(cuda_lib, case):
    """Continuous values: 3xTF32 keeps every element within the fp32 tolerance rule."""
    spc = cuda_lib
    _, dims, B, ci, co, ks, rd, rf = case
    x = uniform_map(B, ci, dims, rd, 4000 + len(dims))
    w = sparse_filter(ci, co, ks, rf, 4001)
    bias = bias_vector(co, 4002)
    V = int(np.prod(dims))
    k = max(1, V // 20)
    fk, fv, fa, _ = ora.conv_fwd(x, w, bias, with_abs=True)
    gk, gv, _ = run_fwd(spc, x, w, bias, "none", k, variant="gemm")
    np.testing.assert_array_equal(gk, fk)
    assert_values_close(gv, fv, fa)
    ok_, ov, _, _ = ora.conv_fwd(x, w, bias, attn=ora.ATTN_MAGNITUDE, k=k)
    gk, gv, _ = run_fwd(spc, x, w, bias, "magnitude", k, variant="gemm")
    assert_topk_sets_match(gk, gv, ok_, ov, fk, fv, fa, V, k, "magnitude")


def test_fwd_variant_measure_and_auto(cuda_lib):
    """Per-layer variant choice by measurement agrees with both variants' results."""
    spc = cuda_lib
    x = uniform_map(1, 16, (8, 8, 32), 0.2, 55, values="dyadic")
    w = sparse_filter(16, 16, (3, 3, 3), 1.0, 56, values="dyadic4")
    X, W = dev_map(spc, x), dev_filter(spc, w)
    k = 100
    ys = {v: spc.sparse_conv_fwd(X, W, None, "magnitude", k, variant=v).trimmed() for v in ("scatter", "gemm", "auto")}
    choice = spc.ops.select_variant(X, W, None, "magnitude", k)
    assert choice in ("scatter", "gemm")
    ym = spc.sparse_conv_fwd(X, W, None, "magnitude", k, variant="measure").trimmed()
    for v in list(ys.values()) + [ym]:
        assert torch.equal(v[0], ys["scatter"][0]) and torch.equal(v[1], ys["scatter"][1])


def test_fwd_gemm_empty_and_unsupported(cuda_lib):
    spc = cuda_lib
    x = COO(2, 2, (5, 6), np.zeros(0, np.uint64), np.zeros(0, np.float32))
    w = sparse_filter(2, 3, (3, 3), 0.5, 3)
    gk, _, _ = run_fwd(spc, x, w, None, "magnitude", 4, variant="gemm")
    assert gk.size == 0
    x = uniform_map(2, 2, (5, 6), 0.3, 4)
    w0 = Filter(2, 3, (3, 3), np.zeros(0, np.uint64), np.zeros(0, np.float32))
    gk, _, _ = run_fwd(spc, x, w0, None, "none", 0, variant="gemm")
    assert gk.size == 0
    x = uniform_map(1, 40, (4, 4, 4), 0.2, 5)          # c_in > 32: G unsupported, explicit request fails
    w = sparse_filter(40, 4, (3, 3, 3), 0.5, 6)
    with pytest.raises(spc.SpconvError):
        run_fwd(spc, x, w, None, "none", 0, variant="gemm")
    gk, _, _ = run_fwd(spc, x, w, None, "none", 0, variant="auto")   # AUTO falls back to S
    assert gk.size > 0


def test_fwd_mnist_like_c1(cuda_lib):
    """BASELINE configs[0]: 2D 28x28, 1->8, 3x3, rho_up 15%, batch 4 (k = floor(0.15*784))."""
    spc = cuda_lib
    x = mnist_like(4, SEED_BASE, values="dyadic")
    w = sparse_filter(1, 8, (3, 3), 1.0, SEED_BASE, values="dyadic")
    bias = bias_vector(8, SEED_BASE, values="dyadic")
    k = int(0.15 * 784)
    ok_, ov, _, _ = ora.conv_fwd(x, w, bias, attn=ora.ATTN_MAGNITUDE, k=k)
    gk, gv, _ = run_fwd(spc, x, w, bias, "magnitude", k)
    np.testing.assert_array_equal(gk, ok_)
    np.testing.assert_array_equal(gv, ov)


def test_fwd_binary_surface_ties(cuda_lib):
    """Binary occupancy (value 1.0): massive exact ties at the threshold (reading R7)."""
    spc = cuda_lib
    x = surface_occupancy(2, 24, 0.05, 77)
    w = sparse_filter(1, 4, (3, 3, 3), 1.0, 77, values="dyadic")
    k = int(0.05 * 24 ** 3)
    for attn in ("magnitude", "raw"):
        ok_, ov, _, _ = ora.conv_fwd(x, w, None, attn=ATTN_ORA[attn], k=k)
        gk, gv, _ = run_fwd(spc, x, w, None, attn, k)
        np.testing.assert_array_equal(gk, ok_)
        np.testing.assert_array_equal(gv, ov)


# Segments large enough for the streamed forward's sampled threshold (>= 34 tiles per segment):
# the candidates (score >= the sampled tlow) must contain the exact top-k; ragged Z (not a
# multiple of 4) takes the scalar epilogue; 12 output channels = two channel groups.
SAMPLED_CASES = [
    ("3d_sampled", (40, 96, 64), 1, 4, 4, (3, 3, 3), 0.03, 0.5),
    ("3d_sampled_ragged_z", (45, 70, 37), 1, 3, 8, (3, 3, 3), 0.04, 0.5),
    ("3d_sampled_two_groups", (36, 64, 32), 2, 3, 12, (3, 3, 3), 0.05, 0.5),
    ("3d_sampled_z128", (24, 40, 128), 1, 3, 5, (3, 3, 3), 0.03, 0.5),   # full 128-voxel epilogue slots
    ("3d_sampled_z256", (12, 30, 256), 1, 2, 4, (3, 3, 3), 0.03, 0.5),
]


@pytest.mark.parametrize("case", SAMPLED_CASES, ids=lambda c: c[0])
@pytest.mark.parametrize("attn", ["magnitude", "raw"])
@pytest.mark.parametrize("values", ["dyadic", "continuous"])
def test_fwd_sampled_threshold(cuda_lib, case, attn, values):
    spc = cuda_lib
    _, dims, B, ci, co, ks, rd, rf = case
    x = uniform_map(B, ci, dims, rd, 4100, values=values)
    w = sparse_filter(ci, co, ks, rf, 4101, values=values)
    bias = bias_vector(co, 4102, values=values)
    V = int(np.prod(dims))
    k = V // 20
    ok_, ov, _, _ = ora.conv_fwd(x, w, bias, attn=ATTN_ORA[attn], k=k)
    gk, gv, _ = run_fwd(spc, x, w, bias, attn, k)
    if values == "dyadic":
        np.testing.assert_array_equal(gk, ok_)
        np.testing.assert_array_equal(gv, ov)
    else:
        fk, fv, fa, _ = ora.conv_fwd(x, w, bias, with_abs=True)
        assert_topk_sets_match(gk, gv, ok_, ov, fk, fv, fa, V, k, attn)


@pytest.mark.parametrize("attn", ["magnitude", "raw", "none"])
def test_fwd_forced_redo(cuda_lib, monkeypatch, attn):
    """Every segment's sampled threshold forced above all scores (SPC_FWD_FORCE_REDO=1): the
    resolve stage must detect that the candidates miss the k-th response and the redo pass must
    recompute those segments with every support entry as a candidate -- same exact result."""
    spc = cuda_lib
    monkeypatch.setenv("SPC_FWD_FORCE_REDO", "1")
    for dims, B, ci, co in [((40, 96, 64), 2, 3, 4), ((9, 7, 11), 3, 2, 5), ((28, 28), 4, 1, 8)]:
        x = uniform_map(B, ci, dims, 0.05, 4200, values="dyadic")
        w = sparse_filter(ci, co, (3,) * len(dims), 0.6, 4201, values="dyadic")
        bias = bias_vector(co, 4202, values="dyadic")
        V = int(np.prod(dims))
        k = max(1, V // 20)
        ok_, ov, _, _ = ora.conv_fwd(x, w, bias, attn=ATTN_ORA[attn], k=k)
        gk, gv, _ = run_fwd(spc, x, w, bias, attn, k)
        np.testing.assert_array_equal(gk, ok_)
        np.testing.assert_array_equal(gv, ov)


@pytest.mark.parametrize("dims", [(32, 32), (25, 41), (4, 16, 16)], ids=["V1024", "V1025", "3d_V1024"])
@pytest.mark.parametrize("attn", ["magnitude", "raw"])
def test_fwd_resolve_small_segment_boundary(cuda_lib, dims, attn):
    """Segments of <= 1024 voxels are resolved one warp per segment, larger ones one block per
    segment: both sides of the boundary, k from 1 to nearly the whole support, dense and sparse
    inputs -- bit-exact against the oracle."""
    spc = cuda_lib
    V = int(np.prod(dims))
    for rd, k in [(0.3, 1), (0.3, V // 7), (0.05, V // 3), (0.9, V - 3)]:
        x = uniform_map(3, 2, dims, rd, 4300 + k, values="dyadic")
        w = sparse_filter(2, 5, (3,) * len(dims), 0.6, 4301, values="dyadic")
        bias = bias_vector(5, 4302, values="dyadic")
        ok_, ov, _, _ = ora.conv_fwd(x, w, bias, attn=ATTN_ORA[attn], k=k)
        gk, gv, _ = run_fwd(spc, x, w, bias, attn, k)
        np.testing.assert_array_equal(gk, ok_)
        np.testing.assert_array_equal(gv, ov)


@pytest.mark.parametrize("dims,ci", [((40000,), 40), ((2, 30000), 36)])
def test_fwd_bwd_long_rows(cuda_lib, dims, ci):
    """Rows longer than the two-CTAs-per-SM accumulator (1D signals, a long last dimension) with
    more than 32 input channels (no tensor-core variant): the scatter forward takes one CTA per SM
    with the whole shared memory; forward (attention) and backward bit-exact on dyadic data. The
    backward's gradient slab holds ky rows of Z + 2hz columns: a 2D map with 30 k-column rows
    exceeds shared memory and is refused (SPC_ERR_UNSUPPORTED, documented in spconv.h)."""
    spc = cuda_lib
    x = uniform_map(2, ci, dims, 0.004, 7100, values="dyadic")
    w = sparse_filter(ci, 3, (3,) * len(dims), 0.5, 7101, values="dyadic4")
    bias = bias_vector(3, 7102, values="dyadic")
    V = int(np.prod(dims))
    k = V // 30
    ok_, ov, _, _ = ora.conv_fwd(x, w, bias, attn=ora.ATTN_MAGNITUDE, k=k)
    gk, gv, y = run_fwd(spc, x, w, bias, "magnitude", k)
    np.testing.assert_array_equal(gk, ok_)
    np.testing.assert_array_equal(gv, ov)
    dy = grad_values(gk.shape[0], 7103, values="dyadic")
    if len(dims) > 1:
        with pytest.raises(spc.SpconvError):
            spc.sparse_conv_bwd(dev_map(spc, x), dev_filter(spc, w), y.exact(), torch.from_numpy(dy).cuda())
        return
    gdx, gdw, _ = spc.sparse_conv_bwd(dev_map(spc, x), dev_filter(spc, w), y.exact(), torch.from_numpy(dy).cuda())
    odx, odw, _, _, _ = ora.conv_bwd(x, w, ok_, dy, with_abs=True)
    np.testing.assert_array_equal(host(gdx), odx)
    np.testing.assert_array_equal(host(gdw), odw)


def test_fwd_empty_and_degenerate(cuda_lib):
    spc = cuda_lib
    x = COO(2, 2, (5, 6), np.zeros(0, np.uint64), np.zeros(0, np.float32))
    w = sparse_filter(2, 3, (3, 3), 0.5, 3)
    gk, gv, y = run_fwd(spc, x, w, None, "magnitude", 4)
    assert gk.size == 0
    # empty filter
    x = uniform_map(2, 2, (5, 6), 0.3, 4)
    w0 = Filter(2, 3, (3, 3), np.zeros(0, np.uint64), np.zeros(0, np.float32))
    gk, _, _ = run_fwd(spc, x, w0, None, "none", 0)
    assert gk.size == 0
    # k >= V: identity on the support
    w = sparse_filter(2, 3, (3, 3), 0.5, 3)
    fk, fv, _, _ = ora.conv_fwd(x, w, None)
    gk, gv, _ = run_fwd(spc, x, w, None, "magnitude", 10 ** 6)
    np.testing.assert_array_equal(gk, fk)
    # a stored 0.0 input stays structurally present (reading R3)
    xz = COO(1, 1, (5,), np.array([2], np.uint64), np.array([0.0], np.float32))
    wz = Filter(1, 1, (3,), np.arange(3, dtype=np.uint64), np.ones(3, np.float32))
    gk, gv, _ = run_fwd(spc, xz, wz, None, "none", 0)
    assert gk.tolist() == [1, 2, 3] and not gv.any()


def test_fwd_device_nnz_input(cuda_lib):
    """Input with a device nnz word and a larger host bound (chained layers, no host sync)."""
    spc = cuda_lib
    x = uniform_map(2, 2, (9, 10, 11), 0.1, 5, values="dyadic")
    w = sparse_filter(2, 3, (3, 3, 3), 0.5, 5, values="dyadic")
    d = dev_map(spc, x)
    pad = 1000
    keys = torch.cat([d.keys, torch.full((pad,), 2 ** 62, dtype=torch.int64, device="cuda")])
    vals = torch.cat([d.values, torch.ones(pad, device="cuda")])
    nnz = torch.tensor([x.nnz], dtype=torch.int64, device="cuda")
    dd = spc.SparseMap(keys, vals, d.batch, d.channels, d.dims, x.nnz + pad, nnz)
    y = spc.sparse_conv_fwd(dd, dev_filter(spc, w), None, "magnitude", 50)
    yk, yv = y.trimmed()
    ok_, ov, _, _ = ora.conv_fwd(x, w, None, attn=ora.ATTN_MAGNITUDE, k=50)
    np.testing.assert_array_equal(host_keys(yk), ok_)
    np.testing.assert_array_equal(host(yv), ov)


# ----------------------------------------------------------------------------- backward
BWD_CASES = [
    ("2d", (12, 11), 2, 2, 3, (3, 3), 0.2, 0.6),
    ("3d", (10, 9, 12), 2, 3, 4, (3, 3, 3), 0.06, 0.5),
    ("3d_tiles", (20, 24, 36), 2, 8, 8, (3, 3, 3), 0.03, 0.5),
    ("3d_wide_oc", (8, 9, 10), 1, 2, 40, (3, 3, 3), 0.06, 0.4),
    ("1d_k5", (50,), 3, 2, 2, (5,), 0.2, 0.8),
    ("3d_wide_ic", (6, 7, 9), 1, 40, 3, (3, 3, 3), 0.05, 0.3),    # c_in > 32: shared chunk prefix
    ("c5_like", (8, 10, 24), 1, 32, 32, (3, 3, 3), 0.2, 1.0),     # 32 channels, many chunks per ic
]


@pytest.mark.parametrize("case", BWD_CASES, ids=lambda c: c[0])
@pytest.mark.parametrize("values", ["dyadic", "continuous"])
def test_bwd_parity(cuda_lib, case, values):
    spc = cuda_lib
    _, dims, B, ci, co, ks, rd, rf = case
    x = uniform_map(B, ci, dims, rd, 3000, values=values)
    w = sparse_filter(ci, co, ks, rf, 3001, values=values)
    bias = bias_vector(co, 3002, values=values)
    V = int(np.prod(dims))
    k = max(1, V // 10)
    yk, yv, _, _ = ora.conv_fwd(x, w, bias, attn=ora.ATTN_MAGNITUDE, k=k)   # kept keys (oracle)
    dy = grad_values(yk.shape[0], 3003, values=values)
    dx, dw, db, dxa, dwa = ora.conv_bwd(x, w, yk, dy, with_abs=True)
    X, W = dev_map(spc, x), dev_filter(spc, w)
    Y = spc.SparseMap.from_arrays(yk, yv, B, co, dims)
    gdx, gdw, gdb = spc.sparse_conv_bwd(X, W, Y, torch.from_numpy(dy).cuda())
    gdx, gdw, gdb = host(gdx), host(gdw), host(gdb)
    if values == "dyadic":
        np.testing.assert_array_equal(gdx, dx)
        np.testing.assert_array_equal(gdw, dw)
        np.testing.assert_array_equal(gdb, db)
    else:
        assert_values_close(gdx, dx, dxa, "dx")
        assert_values_close(gdw, dw, dwa, "dw")
        assert_values_close(gdb, db, np.full(co, np.abs(dy).sum()), "dbias")
    # separate entry points agree with the oracle too (dx sums over several output-channel
    # groups with fp32 atomics when c_out > 16, so run-to-run bits may differ there)
    gdx2 = host(spc.sparse_conv_bwd_input(X, W, Y, torch.from_numpy(dy).cuda()))
    gdw2, gdb2 = spc.sparse_conv_bwd_weight(X, W, Y, torch.from_numpy(dy).cuda())
    assert_values_close(gdx2, dx, dxa, "dx (bwd_input)")
    assert_values_close(host(gdw2), dw, dwa, "dw (bwd_weight)")
    if values == "dyadic" or co <= 16:
        np.testing.assert_array_equal(gdx2, gdx)
    np.testing.assert_array_equal(host(gdb2), gdb)


def test_bwd_zero_dy_and_empty(cuda_lib):
    spc = cuda_lib
    x = uniform_map(2, 2, (7, 8), 0.3, 9)
    w = sparse_filter(2, 2, (3, 3), 0.5, 9)
    yk, yv, _, _ = ora.conv_fwd(x, w, None)
    Y = spc.SparseMap.from_arrays(yk, yv, 2, 2, (7, 8))
    gdx, gdw, gdb = spc.sparse_conv_bwd(dev_map(spc, x), dev_filter(spc, w), Y,
                                        torch.zeros(yk.shape[0], device="cuda"))
    assert not host(gdx).any() and not host(gdw).any() and not host(gdb).any()
    Ye = spc.SparseMap.from_arrays(np.zeros(0, np.uint64), np.zeros(0, np.float32), 2, 2, (7, 8))
    gdx, gdw, gdb = spc.sparse_conv_bwd(dev_map(spc, x), dev_filter(spc, w), Ye, torch.zeros(1, device="cuda"))
    assert not host(gdx).any() and not host(gdw).any() and not host(gdb).any()


# ----------------------------------------------------------------------- other layers
@pytest.mark.parametrize("attn", ["magnitude", "raw"])
def test_topk_parity(cuda_lib, attn):
    spc = cuda_lib
    x = uniform_map(3, 4, (11, 13, 9), 0.3, 41, values="dyadic")   # many exact ties
    k = 37
    ok_, ov, osrc = ora.topk(x, ATTN_ORA[attn], k)
    y, src = spc.attention_topk(dev_map(spc, x), attn, k)
    yk, yv = y.trimmed()
    n = yk.shape[0]
    np.testing.assert_array_equal(host_keys(yk), ok_)
    np.testing.assert_array_equal(host(yv), ov)
    np.testing.assert_array_equal(host(src[:n]), osrc)


def test_topk_large_segments(cuda_lib):
    spc = cuda_lib
    x = uniform_map(2, 2, (64, 64, 16), 0.2, 43)   # segments of 13k entries, several chunks
    k = 2000
    ok_, ov, osrc = ora.topk(x, ora.ATTN_MAGNITUDE, k)
    y, src = spc.attention_topk(dev_map(spc, x), "magnitude", k)
    yk, yv = y.trimmed()
    np.testing.assert_array_equal(host_keys(yk), ok_)
    np.testing.assert_array_equal(host(yv), ov)
    np.testing.assert_array_equal(host(src[:yk.shape[0]]), osrc)


@pytest.mark.parametrize("attn", ["magnitude", "raw"])
@pytest.mark.parametrize("values", ["continuous", "ties"])
def test_topk_13bit_digit_segments(cuda_lib, attn, values):
    """Segments of >= 32 Ki entries take the 13-bit first digit (topk_bits): continuous values
    with k near half the segment (the bench's shape: the threshold bucket holds thousands of
    candidates), and massive ties (+-1, +0, -0) where whole buckets straddle k."""
    spc = cuda_lib
    x = uniform_map(1, 3, (64, 64, 64), 0.2, 47)    # ~52 k entries per segment
    if values == "ties":
        rng = np.random.default_rng(47)
        vals = np.where(rng.random(x.nnz) < 0.5, 1.0, -1.0).astype(np.float32)
        vals[rng.random(x.nnz) < 0.1] = 0.0
        vals[rng.random(x.nnz) < 0.1] = -0.0
        x = COO(x.batch, x.channels, x.dims, x.keys, vals)
    for k in (1, 999, 26000, 51000):
        ok_, ov, osrc = ora.topk(x, ATTN_ORA[attn], k)
        y, src = spc.attention_topk(dev_map(spc, x), attn, k)
        yk, yv = y.trimmed()
        np.testing.assert_array_equal(host_keys(yk), ok_)
        np.testing.assert_array_equal(host(yv).view(np.uint32), ov.view(np.uint32))
        np.testing.assert_array_equal(host(src[:yk.shape[0]]), osrc)


def test_relu_parity(cuda_lib):
    spc = cuda_lib
    for x in [uniform_map(3, 5, (17, 19), 0.3, 51), uniform_map(1, 1, (10,), 0.0, 1),
              uniform_map(2, 3, (40, 40, 10), 0.2, 52)]:
        ok_, ov, osrc = ora.relu(x)
        y, src = spc.sparse_relu(dev_map(spc, x))
        yk, yv = y.trimmed()
        np.testing.assert_array_equal(host_keys(yk), ok_)
        np.testing.assert_array_equal(host(yv), ov)
        np.testing.assert_array_equal(host(src[:yk.shape[0]]), osrc)


@pytest.mark.parametrize("dims,stride,density", [
    ((28, 28), (2, 2), 0.3), ((7, 9), (2, 3), 0.3), ((16, 16, 16), (2, 2, 2), 0.3),
    ((5, 7, 1100), (2, 3, 2), 0.3), ((30,), (4,), 0.3),
    ((3, 9000), (1, 2), 0.3),                 # PZ > 4096: row form
    ((5, 21, 3000), (2, 2, 2), 0.1),          # tile form, several bands per plane, ragged band
    ((9, 11, 13), (3, 1, 4), 0.9),            # dense, ragged windows in every dim
    ((33, 32, 31), (2, 2, 2), 0.05),          # C4-like density
])
def test_maxpool_parity(cuda_lib, dims, stride, density):
    spc = cuda_lib
    x = uniform_map(2, 3, dims, density, 61, values="dyadic")   # exact ties exercise the argmax rule
    ok_, ov, oarg = ora.maxpool(x, stride)
    y, arg = spc.sparse_maxpool(dev_map(spc, x), stride)
    yk, yv = y.trimmed()
    np.testing.assert_array_equal(host_keys(yk), ok_)
    np.testing.assert_array_equal(host(yv), ov)
    np.testing.assert_array_equal(host(arg[:yk.shape[0]]), oarg)


@pytest.mark.parametrize("dims,stride", [((16, 16, 16), (2, 2, 2)), ((9, 11, 13), (3, 1, 4)), ((28, 28), (2, 2))])
def test_maxpool_signed_zero_ties(cuda_lib, dims, stride):
    """Members drawn from {-1, -0.5, -0, +0, +0.5} at high density: +0 and -0 compare equal
    (reading R8: max over stored entries, ties -> smaller input key), so the maximum's value and
    its argmax come from the first member of a cluster's tied zeros (the +0 / -0 branch)."""
    spc = cuda_lib
    x = uniform_map(2, 3, dims, 0.8, 62, values="signed_zero")
    ok_, ov, oarg = ora.maxpool(x, stride)
    y, arg = spc.sparse_maxpool(dev_map(spc, x), stride)
    yk, yv = y.trimmed()
    np.testing.assert_array_equal(host_keys(yk), ok_)
    np.testing.assert_array_equal(host(yv).view(np.uint32), ov.view(np.uint32))   # the sign of zero too
    np.testing.assert_array_equal(host(arg[:yk.shape[0]]), oarg)
    assert np.any(ov == 0) and np.any(np.signbit(ov[ov == 0]))   # the -0 branch was exercised


def test_scatter_grad_parity(cuda_lib):
    spc = cuda_lib
    x = uniform_map(2, 3, (9, 9), 0.4, 71)
    _, _, src = ora.relu(x)
    dy = grad_values(src.shape[0], 71)
    want = ora.scatter_grad(src, dy, x.nnz)
    got = spc.sparse_scatter_grad(torch.from_numpy(src).cuda(), torch.from_numpy(dy).cuda(), src.shape[0], x.nnz)
    np.testing.assert_array_equal(host(got), want)


@pytest.mark.parametrize("case", ["relu", "topk", "sparse_tail", "empty", "bound"])
def test_scatter_grad_sorted_parity(cuda_lib, case):
    """sparse_scatter_grad_sorted (Eq. (5) with key-ordered sources): bit-exact vs the oracle,
    including long zero gaps (warp-cooperative fill), an empty source list, and a device count
    below the bound."""
    spc = cuda_lib
    x = uniform_map(2, 3, (17, 19), 0.4, 73)
    if case in ("relu", "bound"):
        _, _, src = ora.relu(x)
    elif case == "topk":
        _, _, src = ora.topk(x, ora.ATTN_MAGNITUDE, 20)
    elif case == "sparse_tail":
        src = np.array([3, 5, 300, 301, x.nnz - 200], dtype=np.int64)
    else:
        src = np.zeros(0, dtype=np.int64)
    dy = grad_values(max(src.shape[0], 1), 73)[:src.shape[0]]
    n_use = src.shape[0] if case != "bound" else src.shape[0] // 2
    want = ora.scatter_grad(src[:n_use], dy[:n_use], x.nnz)
    s_dev = torch.from_numpy(np.concatenate([src, np.zeros(1, np.int64)])).cuda()
    d_dev = torch.from_numpy(np.concatenate([dy, np.zeros(1, np.float32)])).cuda()
    n_dev = torch.tensor([n_use], dtype=torch.int64, device="cuda") if case == "bound" else None
    got = spc.sparse_scatter_grad(s_dev, d_dev, src.shape[0], x.nnz, n_out_dev=n_dev, sorted=True)
    np.testing.assert_array_equal(host(got), want)


@pytest.mark.parametrize("batch", [16, pytest.param(256, marks=pytest.mark.slow)])
def test_chain_c2_like_device_nnz(cuda_lib, batch):
    """BASELINE configs[1] (batch 256: the full size; 16 in the quick suite): 3 x [conv+attention
    -> ReLU -> maxpool2], 1->8->16->32, chained on the device with no host sync between layers.
    Dyadic values on coarsening grids; the oracle certifies (sum|terms| * 2^e < 2^24) that blocks
    1-2 are exact in fp32 in any order, so they must match bit for bit; block 3 is compared with
    the tolerance rule."""
    spc = cuda_lib
    x = mnist_like(batch, SEED_BASE + 1, values="dyadic")
    chans = [1, 8, 16, 32]
    ks = [117, 29, 7]
    ws = [sparse_filter(1, 8, (3, 3), 1.0, 80, values="dyadic", scale=0.25),
          sparse_filter(8, 16, (3, 3), 1.0, 81, values="dyadic4", scale=0.125),
          sparse_filter(16, 32, (3, 3), 1.0, 82, values="dyadic4", scale=0.125)]
    bs = [bias_vector(chans[i + 1], 90 + i, values="dyadic") for i in range(3)]
    grid_e = [14, 19, 24]
    g = dev_map(spc, x)
    cur = x
    for i in range(3):
        yk, yv, ya, _ = ora.conv_fwd(cur, ws[i], bs[i], attn=ora.ATTN_MAGNITUDE, k=ks[i], with_abs=True)
        g = spc.sparse_conv_fwd(g, dev_filter(spc, ws[i]), torch.from_numpy(bs[i]).cuda(), "magnitude", ks[i])
        gk, gv = g.trimmed()
        if i < 2:
            assert np.all(ya * 2.0 ** grid_e[i] < 2.0 ** 24)     # exactness certificate
            np.testing.assert_array_equal(host_keys(gk), yk)
            np.testing.assert_array_equal(host(gv), yv)
        else:
            fk, fv, fa, _ = ora.conv_fwd(cur, ws[i], bs[i], with_abs=True)
            assert_topk_sets_match(host_keys(gk), host(gv), yk, yv, fk, fv, fa, 49, ks[i], "magnitude")
            return
        cur = COO(cur.batch, chans[i + 1], cur.dims, yk, yv)
        rk, rv, _ = ora.relu(cur)
        cur = COO(cur.batch, chans[i + 1], cur.dims, rk, rv)
        pk, pv, _ = ora.maxpool(cur, (2, 2))
        cur = COO(cur.batch, chans[i + 1], tuple(-(-d // 2) for d in cur.dims), pk, pv)
        g, _ = spc.sparse_relu(g)
        g, _ = spc.sparse_maxpool(g, (2, 2))
        gk, gv = g.trimmed()
        np.testing.assert_array_equal(host_keys(gk), cur.keys)
        np.testing.assert_array_equal(host(gv), cur.values)


# ------------------------------------------------------------------------------ errors
def test_error_codes(cuda_lib):
    spc = cuda_lib
    from paper_1801_10585_b200._lib import SpconvError
    import ctypes as C

    x = uniform_map(1, 2, (6, 6), 0.3, 3)
    w = sparse_filter(2, 2, (3, 3), 0.5, 3)
    X, W = dev_map(spc, x), dev_filter(spc, w)
    plan = spc.FwdPlan(X, W, "magnitude", 5)
    plan.out.capacity = 3
    with pytest.raises(SpconvError) as e:
        plan(X, W)
    assert e.value.code == 3
    plan.out.capacity = plan.capacity
    small = plan.ws[:16]
    plan.ws = small
    with pytest.raises(SpconvError) as e:
        plan(X, W)
    assert e.value.code == 4


def test_validate_env_detects_unsorted(cuda_lib, monkeypatch):
    spc = cuda_lib
    from paper_1801_10585_b200._lib import SpconvError

    x = uniform_map(1, 2, (6, 6), 0.5, 3)
    keys = x.keys.copy()
    keys[[1, 2]] = keys[[2, 1]]
    bad = COO(1, 2, (6, 6), keys, x.values)
    monkeypatch.setenv("SPC_VALIDATE", "1")
    with pytest.raises(SpconvError) as e:
        spc.sparse_relu(dev_map(spc, bad))
    assert e.value.code == 5
    spc.sparse_relu(dev_map(spc, x))   # sorted input passes validation


def test_validate_env_detects_bad_filter(cuda_lib, monkeypatch):
    """SPC_VALIDATE=1 also checks the filter keys: an out-of-range or unsorted filter
    is rejected before any table is built; without validation the tables stay in bounds."""
    spc = cuda_lib
    from paper_1801_10585_b200._lib import SpconvError

    x = uniform_map(1, 2, (6, 6), 0.5, 3)
    w = sparse_filter(2, 3, (3, 3), 0.5, 3)
    X = dev_map(spc, x)
    bad_range = Filter(2, 3, (3, 3), np.append(w.keys[:-1], np.uint64(2 * 3 * 9 + 5)), w.values)
    swapped = w.keys.copy()
    swapped[[0, 1]] = swapped[[1, 0]]
    bad_order = Filter(2, 3, (3, 3), swapped, w.values)
    monkeypatch.setenv("SPC_VALIDATE", "1")
    for bad in (bad_range, bad_order):
        with pytest.raises(SpconvError) as e:
            spc.sparse_conv_fwd(X, dev_filter(spc, bad), None, "magnitude", 5)
        assert e.value.code == 5
    spc.sparse_conv_fwd(X, dev_filter(spc, w), None, "magnitude", 5)   # a valid filter passes
    monkeypatch.delenv("SPC_VALIDATE")
    spc.sparse_conv_fwd(X, dev_filter(spc, bad_range), None, "magnitude", 5)   # no fault, result unspecified
    torch.cuda.synchronize()


# ------------------------------------------------------------- full size (bench config)
@pytest.mark.slow
def test_c4_full_size_sampled(cuda_lib):
    """BASELINE configs[3] at full size in the bench launch configuration: 128^3, b=64, 8->8,
    rho_d 2%, rho_f 0.5, rho_up 5%. The GPU runs the whole batch; the oracle recomputes two
    sampled samples (forward and dx are per-sample) on dyadic inputs -> bit-exact; nnz bound
    holds for every (b, oc)."""
    spc = cuda_lib
    import bench

    cfg = bench.c4_inputs(density=0.02, values="dyadic")
    x, w, bias, k = cfg["x"], cfg["w"], cfg["bias"], cfg["k"]
    X, W = dev_map(spc, x), dev_filter(spc, w)
    y = spc.sparse_conv_fwd(X, W, torch.from_numpy(bias).cuda(), "magnitude", k)
    yk, yv = y.trimmed()
    gk, gv = host_keys(yk), host(yv)
    V = 128 ** 3
    seg = (gk // np.uint64(V)).astype(np.int64)
    assert np.bincount(seg, minlength=64 * 8).max() <= k
    dy = grad_values(gk.shape[0], SEED_BASE + 7, values="dyadic")
    gdx, gdw, gdb = spc.sparse_conv_bwd(X, W, spc.SparseMap.from_arrays(gk, gv, 64, 8, (128,) * 3),
                                        torch.from_numpy(dy).cuda())
    gdx = host(gdx)
    span = np.uint64(8 * V)
    for b in (0, 37):
        xs = select_samples(x, [b])
        ok_, ov, _, _ = ora.conv_fwd(xs, w, bias, attn=ora.ATTN_MAGNITUDE, k=k)
        lo, hi = np.searchsorted(gk, np.uint64(b) * span), np.searchsorted(gk, np.uint64(b + 1) * span)
        np.testing.assert_array_equal(gk[lo:hi] - np.uint64(b) * span, ok_)
        np.testing.assert_array_equal(gv[lo:hi], ov)
        odx, _, _, _, _ = ora.conv_bwd(xs, w, ok_, dy[lo:hi])
        xlo, xhi = np.searchsorted(x.keys, np.uint64(b) * span), np.searchsorted(x.keys, np.uint64(b + 1) * span)
        np.testing.assert_array_equal(gdx[xlo:xhi], odx)


@pytest.mark.slow
def test_c4_full_size_continuous_all_samples(cuda_lib):
    """BASELINE configs[3] at full size (128^3, b = 64, 8 -> 8, rho_d 2 %, rho_f 0.5, rho_up 5 %)
    in continuous values, every sample: the oracle runs per sample in worker processes.
    Forward: per (b, oc) equal kept counts, values within the tolerance rule on the common keys,
    and every key in the symmetric difference within the tolerance of the segment's k-th score.
    Backward with the oracle's kept outputs and dy: dx at all 21.5 M inputs and dw / dbias over
    all 64 samples -- the high-contention fp64 reduction -- within the tolerance
    rule (oracle: fp64 per-sample partials added in sample order, rounded once)."""
    spc = cuda_lib
    import bench
    from tests._oracle_pool import per_sample_oracle

    cfg = bench.c4_inputs(density=0.02, values="continuous")
    x, w, bias, k = cfg["x"], cfg["w"], cfg["bias"], cfg["k"]
    o = per_sample_oracle(x, w, bias, ora.ATTN_MAGNITUDE, k, SEED_BASE + 11)
    X, W = dev_map(spc, x), dev_filter(spc, w)
    y = spc.sparse_conv_fwd(X, W, torch.from_numpy(bias).cuda(), "magnitude", k)
    yk, yv = y.trimmed()
    gk, gv = host_keys(yk), host(yv)
    V = 128 ** 3
    nseg = 64 * 8
    ok_, ov, oa = o["yk"], o["yv"], o["ya"]
    gseg, oseg = (gk // np.uint64(V)).astype(np.int64), (ok_ // np.uint64(V)).astype(np.int64)
    np.testing.assert_array_equal(np.bincount(gseg, minlength=nseg), np.bincount(oseg, minlength=nseg))
    common, gi, oi = np.intersect1d(gk, ok_, assume_unique=True, return_indices=True)
    assert_values_close(gv[gi], ov[oi], oa[oi], "forward values")
    # k-th score per segment on both sides; swapped keys must sit at the threshold
    tol_abs = 2 * (1e-5 + 1e-6 * 108 * 1.0 + 1e-6 * 0.1)   # |y| <= ~1 here; A <= 108 |x||w| + |b|
    t_o = np.full(nseg, np.inf)
    np.minimum.at(t_o, oseg, np.abs(ov.astype(np.float64)))
    t_g = np.full(nseg, np.inf)
    np.minimum.at(t_g, gseg, np.abs(gv.astype(np.float64)))
    full = np.bincount(oseg, minlength=nseg) == k
    assert np.all(np.abs(t_o[full] - t_g[full]) <= tol_abs)
    only_g = np.setdiff1d(np.arange(gk.shape[0]), gi, assume_unique=True)
    only_o = np.setdiff1d(np.arange(ok_.shape[0]), oi, assume_unique=True)
    assert only_g.shape == only_o.shape
    assert np.all(np.abs(np.abs(gv[only_g]) - t_o[gseg[only_g]]) <= tol_abs)
    assert np.all(np.abs(np.abs(ov[only_o]) - t_g[oseg[only_o]]) <= tol_abs)
    # backward on the oracle's kept set
    Yo = spc.SparseMap.from_arrays(ok_, ov, 64, 8, (128,) * 3)
    gdx, gdw, gdb = spc.sparse_conv_bwd(X, W, Yo, torch.from_numpy(o["dy"]).cuda())
    assert_values_close(host(gdx), o["dx"], o["dxa"], "dx (all samples)")
    assert_values_close(host(gdw), o["dw64"].astype(np.float32), o["dwa"], "dw (all 64 samples)")
    assert_values_close(host(gdb), o["db64"].astype(np.float32), np.full(8, np.abs(o["dy"]).sum()), "dbias")


@pytest.mark.slow
def test_c3_full_size_chain_sampled(cuda_lib):
    """BASELINE configs[2] at full size in the bench's layer chain: 64^3 surface occupancy 2 %
    (binary), b = 32, conv 1 -> 32 (attention k = 5242) -> ReLU -> conv 32 -> 64 (attention),
    then the backward through both layers (ReLU scatter with key-ordered sources). Dyadic weights
    on coarse grids so that the oracle certifies the forward sums exact in fp32 (any order): two
    sampled samples recomputed by the oracle from the original input match bit for bit in keys
    and values of both layers; dx of the 32 -> 64 layer is exact too, dx of the first layer is
    compared with the tolerance rule."""
    spc = cuda_lib
    V = 64 ** 3
    k = int(0.02 * V)
    x = surface_occupancy(32, 64, 0.02, SEED_BASE * 1000 + 300)
    w1 = sparse_filter(1, 32, (3, 3, 3), 1.0, SEED_BASE + 31, values="dyadic", scale=0.25)
    w2 = sparse_filter(32, 64, (3, 3, 3), 1.0, SEED_BASE + 32, values="dyadic4", scale=0.125)
    b1, b2 = bias_vector(32, SEED_BASE + 31, values="dyadic"), bias_vector(64, SEED_BASE + 32, values="dyadic")
    X = dev_map(spc, x)
    Y1 = spc.sparse_conv_fwd(X, dev_filter(spc, w1), torch.from_numpy(b1).cuda(), "magnitude", k)
    R1, src1 = spc.sparse_relu(Y1)
    Y2 = spc.sparse_conv_fwd(R1, dev_filter(spc, w2), torch.from_numpy(b2).cuda(), "magnitude", k)
    y1k, y1v = (host(t) for t in Y1.trimmed())
    r1k, r1v = (host(t) for t in R1.trimmed())
    y2k, y2v = (host(t) for t in Y2.trimmed())
    y1k, r1k, y2k = y1k.view(np.uint64), r1k.view(np.uint64), y2k.view(np.uint64)
    dy2 = grad_values(y2k.shape[0], SEED_BASE + 33, values="dyadic")
    dR1 = spc.sparse_conv_bwd_input(R1, dev_filter(spc, w2), Y2.exact(), torch.from_numpy(dy2).cuda())
    dY1 = spc.sparse_scatter_grad(src1, dR1, R1.nnz_bound, Y1.nnz_bound, R1.nnz_dev, sorted=True)
    dX = spc.sparse_conv_bwd_input(X, dev_filter(spc, w1), Y1.exact(), dY1[:y1k.shape[0]])
    gdr1, gdx = host(dR1), host(dX)
    sl = lambda keys, b, c: slice(int(np.searchsorted(keys, np.uint64(b * c * V))),
                                  int(np.searchsorted(keys, np.uint64((b + 1) * c * V))))
    for b in (0, 19):
        xs = select_samples(x, [b])
        o1k, o1v, o1a, _ = ora.conv_fwd(xs, w1, b1, attn=ora.ATTN_MAGNITUDE, k=k, with_abs=True)
        assert np.all(o1a * 2.0 ** 8 < 2.0 ** 24)   # exactness certificate (grid 2^-8)
        s1 = sl(y1k, b, 32)
        np.testing.assert_array_equal(y1k[s1] - np.uint64(b * 32 * V), o1k)
        np.testing.assert_array_equal(y1v[s1], o1v)
        ra = COO(1, 32, (64, 64, 64), o1k, o1v)
        ork, orv, osrc = ora.relu(ra)
        sr = sl(r1k, b, 32)
        np.testing.assert_array_equal(r1k[sr] - np.uint64(b * 32 * V), ork)
        rs = COO(1, 32, (64, 64, 64), ork, orv)
        o2k, o2v, o2a, _ = ora.conv_fwd(rs, w2, b2, attn=ora.ATTN_MAGNITUDE, k=k, with_abs=True)
        assert np.all(o2a * 2.0 ** 13 < 2.0 ** 24)   # (grid 2^-13)
        s2 = sl(y2k, b, 64)
        np.testing.assert_array_equal(y2k[s2] - np.uint64(b * 64 * V), o2k)
        np.testing.assert_array_equal(y2v[s2], o2v)
        odr, _, _, odra, _ = ora.conv_bwd(rs, w2, o2k, dy2[s2], with_abs=True)
        assert np.all(odra * 2.0 ** 11 < 2.0 ** 24)
        np.testing.assert_array_equal(gdr1[sr], odr)
        ody1 = ora.scatter_grad(osrc, odr, o1k.shape[0])
        odx, _, _, odxa, _ = ora.conv_bwd(xs, w1, o1k, ody1, with_abs=True)
        sx = sl(x.keys, b, 1)
        assert_values_close(gdx[sx], odx, odxa, f"first-layer dx, sample {b}")


@pytest.mark.slow
def test_c5_full_size_gemm_sampled(cuda_lib):
    """BASELINE configs[4] at full size for variant G (the tensor-core path the per-layer choice
    takes there): 64^3, b=8, 32->32, rho_d 20%, exact layer. Two sampled samples against the
    oracle: identical support, values within the tolerance rule."""
    spc = cuda_lib
    x = uniform_map(8, 32, (64, 64, 64), 0.2, SEED_BASE * 1000 + 520)
    w = sparse_filter(32, 32, (3, 3, 3), 1.0, SEED_BASE + 5)
    bias = bias_vector(32, SEED_BASE + 5)
    gk, gv, _ = run_fwd(spc, x, w, bias, "none", 0, variant="gemm")
    V = 64 ** 3
    span = np.uint64(32 * V)
    for b in (0, 5):
        xs = select_samples(x, [b])
        fk, fv, fa, _ = ora.conv_fwd(xs, w, bias, with_abs=True)
        lo, hi = np.searchsorted(gk, np.uint64(b) * span), np.searchsorted(gk, np.uint64(b + 1) * span)
        np.testing.assert_array_equal(gk[lo:hi] - np.uint64(b) * span, fk)
        assert_values_close(gv[lo:hi], fv, fa)


# ------------------------------------------------------------ training-loop steps
def test_adagrad_step_bit_exact(cuda_lib):
    """The GPU step performs the oracle's sequence of IEEE double operations: bit-identical, with
    and without the density regulariser (rho from the forward output's device count)."""
    spc = cuda_lib
    x = uniform_map(2, 3, (12, 12, 12), 0.05, 901)
    w = sparse_filter(3, 4, (3, 3, 3), 0.5, 902)
    X, W = dev_map(spc, x), dev_filter(spc, w)
    k = 40
    Y = spc.sparse_conv_fwd(X, W, None, "magnitude", k)
    nnz_y = Y.nnz()
    rng = np.random.default_rng(903)
    n = w.values.size
    dw = rng.normal(0, 0.3, n).astype(np.float32)
    acc0 = rng.uniform(0, 0.5, n).astype(np.float32)
    cells = 2 * 4 * 12 ** 3
    for reg in (None, spc.DensityReg(lam=0.2, rho_up=0.01), spc.DensityReg(lam=0.1, rho_up=0.5, o=0.1, b1=0.3, b2=0.2)):
        p = W.values.clone()
        a = torch.from_numpy(acc0).cuda()
        spc.adagrad_step(p, torch.from_numpy(dw).cuda(), a, lr=0.05, eps=1e-8, reg=reg, y=Y)
        b = 0.0 if reg is None else ora.density_bias(nnz_y / cells, reg.rho_up, reg.o, reg.b1, reg.b2)
        ow, oa = ora.adagrad_step(w.values, dw, acc0, b, 0.0 if reg is None else reg.lam, 0.05, 1e-8)
        np.testing.assert_array_equal(host(p), ow)
        np.testing.assert_array_equal(host(a), oa)


def test_filter_prune_bit_exact_over_epochs(cuda_lib):
    """Pruning over several epoch ends (weights shrinking towards 0) matches the oracle exactly,
    and the pruned filter still convolves like the oracle (pruned weights are simply absent)."""
    spc = cuda_lib
    w = sparse_filter(4, 4, (3, 3, 3), 1.0, 911)
    W = dev_filter(spc, w)
    keys, vals = w.keys.copy(), w.values.copy()
    acc = np.random.default_rng(912).uniform(0, 1, vals.size).astype(np.float32)
    warn = np.zeros(vals.size, np.uint8)
    A, WR = torch.from_numpy(acc).cuda(), torch.zeros(vals.size, dtype=torch.uint8, device="cuda")
    rng = np.random.default_rng(913)
    for ep in range(5):
        vals = (vals * rng.uniform(0.2, 1.2, vals.size)).astype(np.float32)
        W = spc.SparseFilter(W.keys, torch.from_numpy(vals).cuda(), W.c_in, W.c_out, W.ksize)
        W, A, WR = spc.filter_prune(W, A, WR, 0.05)
        keys, vals, acc, warn = ora.prune(keys, vals, acc, warn, 0.05)
        np.testing.assert_array_equal(host_keys(W.keys), keys)
        np.testing.assert_array_equal(host(W.values), vals)
        np.testing.assert_array_equal(host(A), acc)
        np.testing.assert_array_equal(host(WR), warn)
    assert keys.size < w.keys.size
    x = uniform_map(1, 4, (10, 10, 10), 0.1, 914)
    wp = Filter(4, 4, (3, 3, 3), keys, vals)
    fk, fv, fa, _ = ora.conv_fwd(x, wp, None, with_abs=True)
    gk, gv, _ = run_fwd(spc, x, wp, None, "none", 0)
    np.testing.assert_array_equal(gk, fk)
    assert_values_close(gv, fv, fa)


# ------------------------------------------------------------ sparseToDense bridge
def test_sparse_to_dense_and_backward(cuda_lib):
    spc = cuda_lib
    for x in (uniform_map(2, 3, (9, 10, 11), 0.1, 71), uniform_map(3, 2, (28, 28), 0.25, 72),
              COO(1, 2, (4, 4), np.zeros(0, np.uint64), np.zeros(0, np.float32))):
        X = dev_map(spc, x)
        d = spc.sparse_to_dense(X)
        np.testing.assert_array_equal(host(d), ora.to_dense(x))
        g = torch.randn_like(d)
        dv = spc.sparse_to_dense_bwd(X, g)
        np.testing.assert_array_equal(host(dv), host(g).reshape(-1)[x.keys.astype(np.int64)])


# ------------------------------------------------------------------ batch-sliced forward (f2)
PASS_CASES = [
    # name, dims, batch, c_in, c_out, ksize, rho_d, rho_f, samples_per_pass
    ("1d_b5_spp2", (37,), 5, 2, 3, (3,), 0.2, 0.7, 2),
    ("2d_b3_spp1", (13, 17), 3, 3, 5, (5, 3), 0.1, 0.8, 1),
    ("3d_tiles_b3_spp2", (24, 20, 40), 3, 8, 8, (3, 3, 3), 0.03, 0.5, 2),
    ("3d_wide_oc_b4_spp3", (10, 12, 14), 4, 2, 40, (3, 3, 3), 0.05, 0.3, 3),
    ("3d_b2_spp_all", (9, 7, 11), 2, 3, 4, (3, 3, 3), 0.08, 0.5, 0),
]


@pytest.mark.parametrize("case", PASS_CASES, ids=lambda c: c[0])
@pytest.mark.parametrize("attn", ["none", "magnitude", "raw"])
def test_fwd_pass_matches_oracle_and_full(cuda_lib, case, attn):
    """sparse_conv_fwd_pass (bounded workspace, ragged last pass): dyadic values bit-exact vs the
    oracle, and identical (keys and value bits) to the one-shot scatter forward."""
    spc = cuda_lib
    _, dims, B, ci, co, ks, rd, rf, spp = case
    x = uniform_map(B, ci, dims, rd, 1500 + B, values="dyadic")
    w = sparse_filter(ci, co, ks, rf, 1501, values="dyadic")
    bias = bias_vector(co, 1502, values="dyadic")
    V = int(np.prod(dims))
    k = max(1, V // 20)
    ok_, ov, _, _ = ora.conv_fwd(x, w, bias, attn=ATTN_ORA[attn], k=k)
    bt = torch.from_numpy(bias).cuda()
    y = spc.sparse_conv_fwd(dev_map(spc, x), dev_filter(spc, w), bt, attn, k, samples_per_pass=spp)
    pk, pv = (host(t) for t in y.trimmed())
    np.testing.assert_array_equal(pk.view(np.uint64), ok_)
    np.testing.assert_array_equal(pv, ov)
    xc = uniform_map(B, ci, dims, rd, 1600 + B)
    wc = sparse_filter(ci, co, ks, rf, 1601)
    full = spc.sparse_conv_fwd(dev_map(spc, xc), dev_filter(spc, wc), bt, attn, k, variant="scatter")
    part = spc.sparse_conv_fwd(dev_map(spc, xc), dev_filter(spc, wc), bt, attn, k, samples_per_pass=spp)
    fk, fv = (host(t) for t in full.trimmed())
    qk, qv = (host(t) for t in part.trimmed())
    np.testing.assert_array_equal(qk, fk)
    np.testing.assert_array_equal(qv.view(np.uint32), fv.view(np.uint32))


def test_fwd_default_plan_bounds_workspace(cuda_lib, monkeypatch):
    """With the workspace budget at ~0 the default plan slices the batch into one-sample passes
    (ops._bounded_pass) and gives the same keys and value bits as the one-shot forward."""
    spc = cuda_lib
    from paper_1801_10585_b200 import ops
    x = uniform_map(3, 2, (10, 11, 12), 0.1, 77)
    w = sparse_filter(2, 4, (3, 3, 3), 0.5, 77)
    bt = torch.from_numpy(bias_vector(4, 77)).cuda()
    full = spc.sparse_conv_fwd(dev_map(spc, x), dev_filter(spc, w), bt, "magnitude", 60, variant="scatter")
    monkeypatch.setattr(ops, "_WS_FRAC", 1e-12)
    plan = ops.FwdPlan(dev_map(spc, x), dev_filter(spc, w), "magnitude", 60, "scatter", bt)
    assert plan.spp == 1
    part = plan(dev_map(spc, x), dev_filter(spc, w), bt)
    fk, fv = (host(t) for t in full.trimmed())
    qk, qv = (host(t) for t in part.trimmed())
    np.testing.assert_array_equal(qk, fk)
    np.testing.assert_array_equal(qv.view(np.uint32), fv.view(np.uint32))


def test_fwd_pass_device_nnz_and_empty(cuda_lib):
    """Chained input (device nnz word, larger bound) and an all-empty batch through the passes."""
    spc = cuda_lib
    x = uniform_map(3, 2, (9, 10, 11), 0.1, 7, values="dyadic")
    w = sparse_filter(2, 3, (3, 3, 3), 0.5, 7, values="dyadic")
    n = x.keys.size
    keys = torch.zeros(n + 50, dtype=torch.int64, device="cuda")
    vals = torch.zeros(n + 50, dtype=torch.float32, device="cuda")
    keys[:n] = torch.from_numpy(x.keys.view(np.int64)).cuda()
    vals[:n] = torch.from_numpy(x.values).cuda()
    xm = spc.SparseMap(keys, vals, x.batch, x.channels, x.dims, n + 50,
                       torch.tensor([n], dtype=torch.int64, device="cuda"))
    y = spc.sparse_conv_fwd(xm, dev_filter(spc, w), None, "magnitude", 40, samples_per_pass=1)
    ok_, ov, _, _ = ora.conv_fwd(x, w, None, attn=ora.ATTN_MAGNITUDE, k=40)
    gk, gv = (host(t) for t in y.trimmed())
    np.testing.assert_array_equal(gk.view(np.uint64), ok_)
    np.testing.assert_array_equal(gv, ov)
    e = COO(3, 2, (5, 6), np.zeros(0, np.uint64), np.zeros(0, np.float32))
    y = spc.sparse_conv_fwd(dev_map(spc, e), dev_filter(spc, sparse_filter(2, 3, (3, 3), 0.5, 3)), None,
                            "magnitude", 4, samples_per_pass=2)
    assert y.nnz() == 0


@pytest.mark.parametrize("dims", [(37,), (8, 8), (5, 6, 7), (3, 4, 5, 6), (1 << 20, 1 << 20)])
def test_key_codec_parity(cuda_lib, dims):
    """spc_encode_keys / spc_decode_keys against the oracle's codec on seeded coordinates (rank
    1..4; the last case has a key space above 2^32: the 64-bit decode), the SPEC example
    (shape {b=2, 4x4, c=3}, index (b=1, x=2, y=3, c=0) -> 59), round trips, and the
    out-of-range flags."""
    spc = cuda_lib
    B, Cc = 3, 4
    rng = np.random.default_rng(5000 + len(dims))
    n = 2000
    coords = np.stack([rng.integers(0, B, n), rng.integers(0, Cc, n)] +
                      [rng.integers(0, d, n) for d in dims], axis=1).astype(np.int64)
    keys = host(spc.encode_keys(torch.from_numpy(coords).cuda(), B, Cc, dims)).view(np.uint64)
    want = np.array([ora.encode_key(tuple(r), dims, Cc) for r in coords[:300]], np.uint64)
    np.testing.assert_array_equal(keys[:300], want)
    back = host(spc.decode_keys(torch.from_numpy(keys.view(np.int64)).cuda(), B, Cc, dims))
    np.testing.assert_array_equal(back, coords)
    for kk in keys[:50]:
        assert tuple(back[np.nonzero(keys == kk)[0][0]]) == ora.decode_key(int(kk), dims, B, Cc)
    bad = coords[:3].copy()
    bad[1, 2] = dims[0]                       # spatial coordinate out of range
    with pytest.raises(ValueError):
        spc.encode_keys(torch.from_numpy(bad).cuda(), B, Cc, dims)
    total = B * Cc * int(np.prod(dims, dtype=object))
    if total < (1 << 63):
        with pytest.raises(ValueError):
            spc.decode_keys(torch.tensor([0, total], dtype=torch.int64).cuda(), B, Cc, dims)


def test_key_codec_spec_example(cuda_lib):
    spc = cuda_lib
    k = spc.encode_keys(torch.tensor([[1, 0, 2, 3], [0, 0, 0, 0]], dtype=torch.int64).cuda(), 2, 3, (4, 4))
    assert host(k).tolist() == [59, 0]
    c = spc.decode_keys(torch.tensor([59], dtype=torch.int64).cuda(), 2, 3, (4, 4))
    assert host(c).tolist() == [[1, 0, 2, 3]]
    assert spc.encode_keys(torch.zeros((0, 4), dtype=torch.int64).cuda(), 2, 3, (4, 4)).numel() == 0


def test_keys_narrow_widen_roundtrip(cuda_lib):
    """Table 1 "Sparse 32" storage: the low words of the keys and back, bit-exact."""
    spc = cuda_lib
    x = uniform_map(4, 3, (24, 20, 40), 0.05, 9)
    m = dev_map(spc, x)
    k32 = spc.keys_narrow(m)
    assert k32.dtype == torch.int32 and k32.numel() == x.keys.size
    np.testing.assert_array_equal(host(k32).view(np.uint32), x.keys.astype(np.uint32))
    back = spc.keys_widen(k32, m.nnz_bound)
    np.testing.assert_array_equal(host_keys(back), x.keys)


@pytest.mark.parametrize("attn", ["magnitude", "raw"])
def test_topk_ties_across_tiles_and_mixed_segments(cuda_lib, attn):
    """All-equal magnitudes (one tie class spanning several 8192-entry tiles: the tie quota is
    carried across tiles in key order), +0/-0 and sign ties, segments below / above k, empty ones."""
    spc = cuda_lib
    x = uniform_map(3, 2, (40, 40, 16), 0.5, 45)
    rng = np.random.default_rng(45)
    vals = np.where(rng.random(x.nnz) < 0.5, 1.0, -1.0).astype(np.float32)
    vals[rng.random(x.nnz) < 0.05] = 0.0
    vals[rng.random(x.nnz) < 0.05] = -0.0
    seg = (x.keys // np.uint64(40 * 40 * 16)).astype(np.int64)
    keep = (seg != 2) & ~((seg == 4) & (rng.random(x.nnz) < 0.995))   # segment 2 empty, segment 4 tiny
    xs = COO(x.batch, x.channels, x.dims, x.keys[keep], vals[keep])
    for k in (1, 37, 9000, 12000):
        ok_, ov, osrc = ora.topk(xs, ATTN_ORA[attn], k)
        y, src = spc.attention_topk(dev_map(spc, xs), attn, k)
        yk, yv = y.trimmed()
        np.testing.assert_array_equal(host_keys(yk), ok_)
        np.testing.assert_array_equal(host(yv).view(np.uint32), ov.view(np.uint32))
        np.testing.assert_array_equal(host(src[:yk.shape[0]]), osrc)


def test_fwd_tiny_values_keep_structural_support(cuda_lib):
    """Inputs below 2^-50 (products underflow to +-0 in fp32): the forward switches to the
    NaN-marker accumulation (value guard, fused with the row index) so every reached voxel stays
    in the support (reading R3); values compare as numbers (0 == -0)."""
    spc = cuda_lib
    x = uniform_map(2, 3, (9, 10, 11), 0.15, 91)
    w = sparse_filter(3, 4, (3, 3, 3), 0.6, 91)
    vals = x.values.copy()
    vals[::3] *= np.float32(1e-30)          # a third of the inputs tiny: products underflow
    xt = COO(x.batch, x.channels, x.dims, x.keys, vals)
    fk, fv, fa, _ = ora.conv_fwd(xt, w, None, with_abs=True)
    gk, gv, _ = run_fwd(spc, xt, w, None, "none", 0)
    np.testing.assert_array_equal(gk, fk)
    assert_values_close(gv, fv, fa)
    for variant in ("scatter",):
        y = spc.sparse_conv_fwd(dev_map(spc, xt), dev_filter(spc, w), None, "none", 0, variant=variant,
                                samples_per_pass=1)
        pk, pv = (host(t) for t in y.trimmed())
        np.testing.assert_array_equal(pk.view(np.uint64), fk)


# --------------------------------------------- 32-bit key storage (Table 1 "Sparse 32")
def _keys_u64(t):
    a = host(t)
    return a.view(np.uint32).astype(np.uint64) if a.dtype == np.int32 else a.view(np.uint64)


@pytest.mark.parametrize("case", [FWD_CASES[4], FWD_CASES[7], SAMPLED_CASES[1], RANK4_CASES[0]], ids=lambda c: c[0])
@pytest.mark.parametrize("attn", ["none", "magnitude"])
def test_fwd_bwd_32bit_keys(cuda_lib, case, attn):
    """Input and output maps with uint32 keys (spc_map_t.key_bits = 32): the forward, the
    backward and the 64 <-> 32-bit conversions give the oracle's result bit for bit."""
    spc = cuda_lib
    _, dims, B, ci, co, ks, rd, rf = case
    x = uniform_map(B, ci, dims, rd, 4700, values="dyadic")
    w = sparse_filter(ci, co, ks, rf, 4701, values="dyadic")
    bias = bias_vector(co, 4702, values="dyadic")
    V = int(np.prod(dims))
    k = max(1, V // 20)
    X32 = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims, key_bits=32)
    assert X32.key_bits == 32
    Y = spc.sparse_conv_fwd(X32, dev_filter(spc, w), torch.from_numpy(bias).cuda(), attn, k, variant="scatter")
    assert Y.key_bits == 32
    yk, yv = Y.trimmed()
    ok_, ov, _, _ = ora.conv_fwd(x, w, bias, attn=ATTN_ORA[attn], k=k)
    np.testing.assert_array_equal(_keys_u64(yk), ok_)
    np.testing.assert_array_equal(host(yv), ov)
    Y64 = spc.sparse_conv_fwd(X32, dev_filter(spc, w), torch.from_numpy(bias).cuda(), attn, k, variant="scatter",
                              key_bits=64)
    np.testing.assert_array_equal(_keys_u64(Y64.trimmed()[0]), ok_)
    dy = grad_values(ok_.shape[0], 4703, values="dyadic")
    odx, odw, odb, _, _ = ora.conv_bwd(x, w, ok_, dy)
    gdx, gdw, gdb = spc.sparse_conv_bwd(X32, dev_filter(spc, w), Y.exact(), torch.from_numpy(dy).cuda())
    np.testing.assert_array_equal(host(gdx), odx)
    np.testing.assert_array_equal(host(gdw), odw)
    np.testing.assert_array_equal(host(gdb), odb)


def test_relu_pool_topk_32bit_keys(cuda_lib):
    spc = cuda_lib
    x = uniform_map(2, 3, (16, 12, 20), 0.3, 4800, values="dyadic")
    X32 = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims, key_bits=32)
    rk, rv, rsrc = ora.relu(x)
    y, src = spc.sparse_relu(X32)
    np.testing.assert_array_equal(_keys_u64(y.trimmed()[0]), rk)
    np.testing.assert_array_equal(host(src[:rk.shape[0]]), rsrc)
    pk, pv, parg = ora.maxpool(x, (2, 3, 2))
    y, arg = spc.sparse_maxpool(X32, (2, 3, 2))
    np.testing.assert_array_equal(_keys_u64(y.trimmed()[0]), pk)
    np.testing.assert_array_equal(host(y.trimmed()[1]), pv)
    np.testing.assert_array_equal(host(arg[:pk.shape[0]]), parg)
    tk, tv, tsrc = ora.topk(x, ora.ATTN_RAW, 23)
    y, src = spc.attention_topk(X32, "raw", 23)
    np.testing.assert_array_equal(_keys_u64(y.trimmed()[0]), tk)
    np.testing.assert_array_equal(host(y.trimmed()[1]), tv)
    # conversions round-trip, sparse_to_dense reads 32-bit keys too
    X64 = X32.to_key_bits(64)
    np.testing.assert_array_equal(_keys_u64(X64.keys), x.keys)
    np.testing.assert_array_equal(host(spc.sparse_to_dense(X32)), host(spc.sparse_to_dense(X64)))


@pytest.mark.parametrize("attn", ["magnitude", "raw"])
def test_fwd_split_resolve_few_segments(cuda_lib, attn):
    """Fewer segments than SMs with more than 4096 candidates per segment: the forward's resolve
    runs split (multi-CTA candidate histogram and collect, then the per-segment select) -- same
    kept set and values as the oracle's sort (R7)."""
    import paper_1801_10585_b200 as spc

    dims = (40, 44, 48)
    x = uniform_map(1, 2, dims, 0.03, 9100, values="dyadic")
    w = sparse_filter(2, 3, (3, 3, 3), 0.5, 9101, values="dyadic")
    bias = bias_vector(3, 9102, values="dyadic")
    k = int(0.06 * np.prod(dims))
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
    W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
    Y = spc.sparse_conv_fwd(X, W, torch.from_numpy(bias).cuda(), attn, k, variant="scatter")
    yk, yv = Y.trimmed()
    a = ora.ATTN_MAGNITUDE if attn == "magnitude" else ora.ATTN_RAW
    ok, ov, _, _ = ora.conv_fwd(x, w, bias, attn=a, k=k)
    assert ok.shape[0] == 3 * k
    assert np.array_equal(yk.cpu().numpy().view(np.uint64), ok)
    assert np.array_equal(yv.cpu().numpy(), ov)

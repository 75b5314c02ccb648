"""Pins of the CPU oracle against things other than itself (runs without a GPU).

Each test names what fixes the expected value: SPEC/PAPER worked examples (tests/golden/),
brute-force dense convolution (torch CPU fp64, a library routine, and a numpy definition),
fp64 autograd, finite differences, full Python sorts, closed forms and invariants.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

import oracle as ora
from synth import COO, Filter, uniform_map, sparse_filter, bias_vector, grad_values, mnist_like
from tests._brute import (coo_to_dense, filter_to_dense, torch_xcorr, shift_xcorr, dense_to_sorted,
                          brute_topk, masked_conv_grads)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
U24 = 2.0 ** -24


def _coo_from_points(dims, entries, batch=1, channels=1):
    V = int(np.prod(dims))
    keys = np.array(sorted(int(np.ravel_multi_index(p, dims)) for p, _ in entries), np.uint64)
    d = {int(np.ravel_multi_index(p, dims)): v for p, v in entries}
    vals = np.array([d[int(k)] for k in keys], np.float32)
    assert V > 0
    return COO(batch, channels, tuple(dims), keys, vals)


# ----------------------------------------------------------------- golden examples
@pytest.mark.parametrize("ex", GOLD["key_codec"], ids=lambda e: e["source"][:6])
def test_key_codec_golden(ex):
    assert ora.encode_key(ex["index"], ex["dims"], ex["channels"]) == ex["key"]
    assert ora.decode_key(ex["key"], ex["dims"], ex["batch"], ex["channels"]) == tuple(ex["index"])


def test_key_codec_roundtrip_vs_numpy():
    rng = np.random.default_rng(0)
    dims, B, Cc = (5, 7, 3), 3, 4
    for _ in range(200):
        idx = [int(rng.integers(B)), int(rng.integers(Cc))] + [int(rng.integers(d)) for d in dims]
        key = ora.encode_key(idx, dims, Cc)
        assert key == int(np.ravel_multi_index(tuple(idx), (B, Cc) + dims))  # library routine
        assert ora.decode_key(key, dims, B, Cc) == tuple(idx)


@pytest.mark.parametrize("ex", GOLD["get_update_id"], ids=lambda e: e["source"][:6])
def test_get_update_id_golden(ex):
    got = ora.get_update_id(ex["id"], ex["fid"], ex["dims"], ex["ksize"])
    assert got == (tuple(ex["uid"]) if ex["uid"] is not None else None)


@pytest.mark.parametrize("ex", GOLD["k_select"], ids=lambda e: e["source"][:6])
def test_kselect_golden(ex):
    x = COO(1, 1, (len(ex["values"]),), np.arange(len(ex["values"]), dtype=np.uint64),
            np.array(ex["values"], np.float32))
    attn = ora.ATTN_RAW if ex["attn"] == "raw" else ora.ATTN_MAGNITUDE
    _, yv, _ = ora.topk(x, attn, ex["k"])
    np.testing.assert_array_equal(np.sort(yv), np.sort(np.array(ex["kept"], np.float32)))


@pytest.mark.parametrize("ex", GOLD["conv"], ids=lambda e: e["source"][:6])
def test_conv_golden(ex):
    dims = tuple(ex["dims"])
    x = _coo_from_points(dims, [(tuple(int(t) for t in k.split(",")), v) for k, v in ex["x"].items()])
    K = int(np.prod(ex["ksize"]))
    w = Filter(1, 1, tuple(ex["ksize"]), np.arange(K, dtype=np.uint64), np.ones(K, np.float32))
    yk, yv, _, _ = ora.conv_fwd(x, w, None)
    want = {int(np.ravel_multi_index(tuple(int(t) for t in k.split(",")), dims)): v for k, v in ex["y"].items()}
    assert yk.tolist() == sorted(want)
    np.testing.assert_array_equal(yv, np.array([want[k] for k in sorted(want)], np.float32))


def test_identity_1x1_conv():
    """1x1 filter with weight 1.0 on the diagonal ic == oc, zero bias -> output == input."""
    x = uniform_map(2, 3, (6, 5), 0.3, 11)
    ks = (1, 1)
    keys = np.array([(oc * 3 + oc) for oc in range(3)], np.uint64)
    w = Filter(3, 3, ks, keys, np.ones(3, np.float32))
    yk, yv, _, _ = ora.conv_fwd(x, w, None)
    np.testing.assert_array_equal(yk, x.keys)
    np.testing.assert_array_equal(yv, x.values)


@pytest.mark.parametrize("ex", GOLD["maxpool"], ids=lambda e: e["source"][:6])
def test_maxpool_golden(ex):
    x = COO(1, 1, tuple(ex["dims"]), np.array([e[0] for e in ex["x"]], np.uint64),
            np.array([e[1] for e in ex["x"]], np.float32))
    yk, yv, am = ora.maxpool(x, ex["stride"])
    assert yk.tolist() == [e[0] for e in ex["y"]]
    assert yv.tolist() == [e[1] for e in ex["y"]]
    assert am.tolist() == ex["argmax"]


@pytest.mark.parametrize("ex", GOLD["relu"], ids=lambda e: e["source"][:6])
def test_relu_golden(ex):
    n = len(ex["values"])
    x = COO(1, 1, (n,), np.arange(n, dtype=np.uint64), np.array(ex["values"], np.float32))
    _, yv, _ = ora.relu(x)
    assert yv.tolist() == ex["kept"]


# --------------------------------------------------------- forward vs brute force
CASES = [
    # ndim dims, batch, c_in, c_out, ksize, rho_d, rho_f
    ((9,), 2, 2, 3, (3,), 0.3, 0.7),
    ((8, 8), 2, 2, 3, (3, 3), 0.2, 0.5),   # S:170 shape
    ((7, 10), 3, 1, 4, (5, 3), 0.15, 0.8),
    ((6, 5, 7), 2, 3, 2, (3, 3, 3), 0.1, 0.5),
    ((5, 6, 4), 1, 2, 2, (1, 3, 5), 0.3, 1.0),
    ((12, 12, 12), 2, 2, 2, (3, 3, 3), 0.03, 0.5),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "x".join(map(str, c[0])) + f"_k{'x'.join(map(str, c[4]))}")
@pytest.mark.parametrize("values", ["continuous", "dyadic"])
def test_fwd_unbounded_vs_dense_xcorr(case, values):
    """Alg. 1 without attention == dense SAME cross-correlation read on the structural support
    (brute force: torch conv fp64 and the numpy shift definition)."""
    dims, B, ci, co, ks, rd, rf = case
    x = uniform_map(B, ci, dims, rd, 100 + len(dims), values=values)
    w = sparse_filter(ci, co, ks, rf, 7, values=values)
    bias = bias_vector(co, 3, values=values)
    yk, yv, ya, macs = ora.conv_fwd(x, w, bias, with_abs=True)
    Xd, Xm = coo_to_dense(x)
    Wd, Wm = filter_to_dense(w)
    Yd = torch_xcorr(Xd, Wd)
    np.testing.assert_allclose(shift_xcorr(Xd, Wd), Yd, rtol=1e-12, atol=1e-12)
    S = torch_xcorr(Xm.astype(np.float64), Wm.astype(np.float64)) > 0.5  # structural support (P1)
    sk, sv = dense_to_sorted(Yd + bias.astype(np.float64).reshape((1, -1) + (1,) * len(dims)), S)
    np.testing.assert_array_equal(yk, sk)
    # one fp64 -> fp32 rounding at most (different summation order in fp64)
    err = np.abs(yv.astype(np.float64) - sv)
    assert np.all(err <= U24 * np.abs(sv) + 1e-12 * ya), err.max()
    if values == "dyadic":
        np.testing.assert_array_equal(yv, sv.astype(np.float32))
    # macs = number of in-bounds (input, weight) pairs (Eq. (1) first term)
    pairs = torch_xcorr(Xm.astype(np.float64), Wm.astype(np.float64)).sum()
    assert macs == int(round(pairs))


def test_fwd_4d_vs_shift_definition():
    x = uniform_map(1, 2, (4, 3, 5, 4), 0.2, 5)
    w = sparse_filter(2, 2, (3, 1, 3, 3), 0.6, 5)
    yk, yv, _, _ = ora.conv_fwd(x, w, None)
    Xd, Xm = coo_to_dense(x)
    Wd, Wm = filter_to_dense(w)
    S = shift_xcorr(Xm.astype(np.float64), Wm.astype(np.float64)) > 0.5
    sk, sv = dense_to_sorted(shift_xcorr(Xd, Wd), S)
    np.testing.assert_array_equal(yk, sk)
    np.testing.assert_allclose(yv, sv, rtol=2 * U24, atol=1e-12)


def test_library_special_case_dense():
    """rho_d = rho_f = 1, no attention, zero bias: equals torch.nn.functional.conv3d (fp64)
    at every grid point."""
    x = uniform_map(2, 2, (5, 4, 6), 1.0, 9)
    w = sparse_filter(2, 3, (3, 3, 3), 1.0, 9)
    yk, yv, _, _ = ora.conv_fwd(x, w, None)
    Y = torch_xcorr(*[coo_to_dense(x)[0], filter_to_dense(w)[0]])
    assert yk.shape[0] == Y.size
    np.testing.assert_allclose(yv, Y.reshape(-1).astype(np.float32), rtol=2 * U24, atol=1e-7)


def test_macs_closed_form_dense():
    """Dense input, dense filter: in-bounds pairs = b*c_in*c_out*prod_d(s_f*n_d - c_d*(c_d+1))."""
    dims, ks = (6, 7, 5), (3, 5, 3)
    B, ci, co = 2, 2, 3
    x = uniform_map(B, ci, dims, 1.0, 4)
    w = sparse_filter(ci, co, ks, 1.0, 4)
    _, _, _, macs = ora.conv_fwd(x, w, None)
    per = 1
    for n, s in zip(dims, ks):
        c = s // 2
        per *= s * n - c * (c + 1)
    assert macs == B * ci * co * per


def test_macs_linear_in_densities():
    """Eq. (1): the MAC term is linear in rho_d and rho_f (expected value; interior-dominated grid)."""
    base = None
    for rd in (0.02, 0.04):
        for rf in (0.25, 0.5):
            x = uniform_map(2, 2, (24, 24, 24), rd, 21)
            w = sparse_filter(2, 2, (3, 3, 3), rf, 21)
            _, _, _, macs = ora.conv_fwd(x, w, None)
            pred = x.nnz * w.nnz / 2  # c_out-average of weights per input channel
            ratio = macs / pred
            base = ratio if base is None else base
            assert abs(ratio - base) < 0.03 * base


def test_fill_in_uniform_3d():
    """Fig. 2: uniform data under a dense 3x3x3 filter fills the interior to
    1 - (1 - rho)^27 (independent positions)."""
    rho = 0.02
    x = uniform_map(1, 1, (40, 40, 40), rho, 31)
    w = sparse_filter(1, 1, (3, 3, 3), 1.0, 31)
    yk, _, _, _ = ora.conv_fwd(x, w, None)
    m = np.zeros(40 ** 3, bool)
    m[yk.astype(np.int64)] = True
    interior = m.reshape(40, 40, 40)[1:-1, 1:-1, 1:-1].mean()
    # sampling without replacement: P(empty neighbourhood) ~ (1 - rho)^27
    assert abs(interior - (1 - (1 - rho) ** 27)) < 0.01


# ------------------------------------------------------------------------ attention
@pytest.mark.parametrize("attn", ["magnitude", "raw"])
@pytest.mark.parametrize("values", ["continuous", "dyadic"])
def test_fused_attention_vs_full_sort(attn, values):
    """Alg. 1 with attention == brute-force full sort of the exact (unbounded) output per (b, oc),
    rule (score desc, key asc) (readings R5-R7); plus the paper's invariants."""
    dims = (10, 9, 8)
    x = uniform_map(2, 2, dims, 0.05, 41, values=values)
    w = sparse_filter(2, 3, (3, 3, 3), 0.5, 41, values=values)
    bias = bias_vector(3, 41, values=values)
    V = int(np.prod(dims))
    k = int(0.05 * V)
    a = ora.ATTN_MAGNITUDE if attn == "magnitude" else ora.ATTN_RAW
    fk, fv, _, _ = ora.conv_fwd(x, w, bias)
    yk, yv, _, _ = ora.conv_fwd(x, w, bias, attn=a, k=k)
    bk, bv = brute_topk(fk, fv, V, k, attn)
    np.testing.assert_array_equal(yk, bk)
    np.testing.assert_array_equal(yv, bv)
    # invariants: nnz(b, oc) <= k (density bound rho_up*V), dominance
    seg = (yk // np.uint64(V)).astype(np.int64)
    assert np.bincount(seg).max() <= k
    sc = (lambda v: np.abs(v)) if attn == "magnitude" else (lambda v: v)
    fseg = (fk // np.uint64(V)).astype(np.int64)
    kept = set(yk.tolist())
    for s in np.unique(fseg):
        m = fseg == s
        keep = np.array([kk in kept for kk in fk[m].tolist()])
        if (~keep).any():
            assert sc(fv[m][keep]).min() >= sc(fv[m][~keep]).max()


def test_attention_k_ge_support_is_identity():
    x = uniform_map(1, 1, (6, 6), 0.1, 5)
    w = sparse_filter(1, 2, (3, 3), 1.0, 5)
    fk, fv, _, _ = ora.conv_fwd(x, w, None)
    yk, yv, _, _ = ora.conv_fwd(x, w, None, attn=ora.ATTN_MAGNITUDE, k=36)
    np.testing.assert_array_equal(fk, yk)
    np.testing.assert_array_equal(fv, yv)


@pytest.mark.parametrize("attn", ["magnitude", "raw"])
def test_topk_standalone_vs_full_sort(attn):
    x = uniform_map(3, 2, (11, 13), 0.4, 8, values="dyadic")  # many exact ties
    V = 11 * 13
    k = 17
    a = ora.ATTN_MAGNITUDE if attn == "magnitude" else ora.ATTN_RAW
    yk, yv, src = ora.topk(x, a, k)
    bk, bv = brute_topk(x.keys, x.values, V, k, attn)
    np.testing.assert_array_equal(yk, bk)
    np.testing.assert_array_equal(yv, bv)
    np.testing.assert_array_equal(x.keys[src], yk)


def test_topk_negative_zero_ties():
    """R7: -0 and +0 are the same score; ties resolved by smaller key."""
    vals = np.array([0.0, -0.0, 1.0, -0.0, 0.0], np.float32)
    vals[1] = -0.0
    x = COO(1, 1, (5,), np.arange(5, dtype=np.uint64), vals)
    yk, _, _ = ora.topk(x, ora.ATTN_MAGNITUDE, 3)
    assert yk.tolist() == [0, 1, 2]
    yk, _, _ = ora.topk(x, ora.ATTN_RAW, 2)
    assert yk.tolist() == [0, 2]


# ------------------------------------------------------------------------ backward
@pytest.mark.parametrize("dims,ks", [((9, 8), (3, 3)), ((6, 5, 7), (3, 3, 3)), ((11,), (5,))])
@pytest.mark.parametrize("values", ["continuous", "dyadic"])
def test_bwd_vs_autograd(dims, ks, values):
    """Alg. 2 / Eqs. (3)-(4) == fp64 autograd of sum_kept dy*y, read at stored inputs/weights
    (P5). dbias == sum of dy per channel."""
    x = uniform_map(2, 2, dims, 0.25, 61, values=values)
    w = sparse_filter(2, 3, ks, 0.6, 61, values=values)
    bias = bias_vector(3, 61, values=values)
    V = int(np.prod(dims))
    yk, yv, _, _ = ora.conv_fwd(x, w, bias, attn=ora.ATTN_MAGNITUDE, k=max(1, V // 4))
    dy = grad_values(yk.shape[0], 61, values=values)
    dx, dw, db, dxa, dwa = ora.conv_bwd(x, w, yk, dy, with_abs=True)
    gX, gW, gb = masked_conv_grads(x, w, bias, yk, dy)
    ref_dx = gX.reshape(-1)[x.keys.astype(np.int64)]
    ref_dw = gW.reshape(-1)[w.keys.astype(np.int64)]
    assert np.all(np.abs(dx - ref_dx) <= U24 * np.abs(ref_dx) + 1e-12 * dxa)
    assert np.all(np.abs(dw - ref_dw) <= U24 * np.abs(ref_dw) + 1e-12 * dwa)
    np.testing.assert_allclose(db, gb, rtol=2 * U24, atol=1e-12)
    if values == "dyadic":
        np.testing.assert_array_equal(dx, ref_dx.astype(np.float32))
        np.testing.assert_array_equal(dw, ref_dw.astype(np.float32))
    # Eq. (3)/(4) masking: the dense autograd gradient is generally nonzero at non-stored inputs,
    # the sparse rule assigns it no storage at all (fixed shape, P:135 (i)).
    assert dx.shape == (x.nnz,) and dw.shape == (w.nnz,)


def test_bwd_finite_differences():
    """Central differences (step 1e-4, rtol 1e-3) of L = sum dy*y (unbounded, so the
    output set is fixed), perturbing only stored entries."""
    x = uniform_map(1, 2, (6, 6), 0.3, 71)
    w = sparse_filter(2, 2, (3, 3), 0.7, 71)
    bias = bias_vector(2, 71)
    yk, _, _, _ = ora.conv_fwd(x, w, bias)
    dy = grad_values(yk.shape[0], 71)
    dx, dw, db, _, _ = ora.conv_bwd(x, w, yk, dy)

    def L(xv, wv, bv):
        xx = COO(x.batch, x.channels, x.dims, x.keys, xv.astype(np.float32))
        ww = Filter(w.c_in, w.c_out, w.ksize, w.keys, wv.astype(np.float32))
        k2, v2, _, _ = ora.conv_fwd(xx, ww, bv.astype(np.float32))
        assert np.array_equal(k2, yk)
        return float(np.dot(v2.astype(np.float64), dy.astype(np.float64)))

    h = 1e-2  # values are O(1); fp32 forward -> use a larger step, relative check below
    for i in range(0, x.nnz, max(1, x.nnz // 10)):
        e = np.zeros(x.nnz)
        e[i] = h
        fd = (L(x.values + e, w.values, bias) - L(x.values - e, w.values, bias)) / (2 * h)
        assert abs(fd - dx[i]) <= 1e-3 * max(1.0, abs(dx[i]))
    for j in range(0, w.nnz, max(1, w.nnz // 10)):
        e = np.zeros(w.nnz)
        e[j] = h
        fd = (L(x.values, w.values + e, bias) - L(x.values, w.values - e, bias)) / (2 * h)
        assert abs(fd - dw[j]) <= 1e-3 * max(1.0, abs(dw[j]))


def test_bwd_zero_dy():
    x = uniform_map(1, 2, (7, 7), 0.3, 3)
    w = sparse_filter(2, 2, (3, 3), 0.5, 3)
    yk, _, _, _ = ora.conv_fwd(x, w, None)
    dx, dw, db, _, _ = ora.conv_bwd(x, w, yk, np.zeros(yk.shape[0], np.float32))
    assert not dx.any() and not dw.any() and not db.any()


def test_bwd_identity_1x1():
    """identity 1x1 -> dx = dy restricted to input keys; dw[diag] = sum val*g."""
    x = uniform_map(2, 2, (5, 5), 0.4, 13)
    w = Filter(2, 2, (1, 1), np.array([0, 3], np.uint64), np.ones(2, np.float32))
    yk, _, _, _ = ora.conv_fwd(x, w, None)
    np.testing.assert_array_equal(yk, x.keys)
    dy = grad_values(yk.shape[0], 13)
    dx, dw, _, _, _ = ora.conv_bwd(x, w, yk, dy)
    np.testing.assert_array_equal(dx, dy)
    V = 25
    ch = ((x.keys // np.uint64(V)) % np.uint64(2)).astype(np.int64)
    for c in range(2):
        want = np.sum(x.values[ch == c].astype(np.float64) * dy[ch == c].astype(np.float64))
        assert abs(dw[c] - want) <= 1e-6 * max(1.0, abs(want))


# ------------------------------------------------------------------- relu and pooling
def test_relu_definition_and_idempotence():
    x = uniform_map(2, 3, (9, 9), 0.3, 17)
    yk, yv, src = ora.relu(x)
    m = x.values > 0
    np.testing.assert_array_equal(yk, x.keys[m])
    np.testing.assert_array_equal(yv, x.values[m])
    np.testing.assert_array_equal(src, np.nonzero(m)[0])
    y = COO(x.batch, x.channels, x.dims, yk, yv)
    yk2, yv2, _ = ora.relu(y)
    np.testing.assert_array_equal(yk2, yk)


@pytest.mark.parametrize("dims,stride", [((8, 8), (2, 2)), ((7, 9), (2, 3)), ((6, 6, 6), (2, 2, 2)), ((5, 7, 4), (2, 3, 2))])
def test_maxpool_vs_dense(dims, stride):
    """§3.3 pooling == dense max-pool (torch, -inf for absent entries, ceil mode) on occupied
    clusters; argmax == brute-force first maximum in key order."""
    x = uniform_map(2, 2, dims, 0.3, 23, values="dyadic")  # dyadic: exact ties occur
    yk, yv, am = ora.maxpool(x, stride)
    Xd, Xm = coo_to_dense(x)
    Xi = np.where(Xm, Xd, -np.inf)
    nd = len(dims)
    pool = {2: torch.nn.functional.max_pool2d, 3: torch.nn.functional.max_pool3d}[nd]
    P = pool(torch.from_numpy(Xi), kernel_size=stride, stride=stride, ceil_mode=True).numpy()
    occ = np.isfinite(P)
    pk, pv = dense_to_sorted(P, occ)
    np.testing.assert_array_equal(yk, pk)
    np.testing.assert_array_equal(yv, pv.astype(np.float32))
    # argmax: smallest input index attaining the cluster max
    V = int(np.prod(dims))
    odims = tuple(-(-d // s) for d, s in zip(dims, stride))
    best = {}
    for i, (kk, v) in enumerate(zip(x.keys.tolist(), x.values.tolist())):
        seg, sp = divmod(kk, V)
        p = np.unravel_index(sp, dims)
        q = tuple(pi // si for pi, si in zip(p, stride))
        pkk = seg * int(np.prod(odims)) + int(np.ravel_multi_index(q, odims))
        if pkk not in best or v > best[pkk][0]:
            best[pkk] = (v, i)
    assert am.tolist() == [best[k][1] for k in yk.tolist()]


def test_scatter_grad():
    src = np.array([4, 0, 2], np.int64)
    dy = np.array([1.5, -2.0, 3.0], np.float32)
    dx = ora.scatter_grad(src, dy, 6)
    assert dx.tolist() == [-2.0, 0.0, 3.0, 0.0, 1.5, 0.0]


# --------------------------------------------------------------------------- inputs
def test_mnist_like_density_matches_paper():
    """thresholded MNIST has mean density 0.23."""
    m = mnist_like(400, 5)
    assert abs(m.nnz / 400 / 784 - 0.23) < 0.02


# ------------------------------------------------------------ training-loop steps
@pytest.mark.parametrize("ex", GOLD["density_bias"], ids=lambda e: e["cite"][:24])
def test_density_bias_golden(ex):
    b = ora.density_bias(ex["rho"], ex["rho_up"], ex["o"], ex["b1"], ex["b2"])
    assert abs(b - ex["b"]) < 1e-12


def test_density_bias_eq6_shape():
    """Eq. (6): continuous from below at rho_up (b -> 0), a jump of o just above it, slopes b1
    above and b2 below (finite differences), positive iff rho > rho_up."""
    o, b1, b2, up = 0.1, 0.3, 0.2, 0.15
    eps = 1e-7
    assert abs(ora.density_bias(up, up, o, b1, b2)) < 1e-15
    assert abs(ora.density_bias(up + eps, up, o, b1, b2) - o) < 1e-6
    for r in (0.3, 0.6):
        assert abs((ora.density_bias(r + 1e-4, up, o, b1, b2) - ora.density_bias(r, up, o, b1, b2)) / 1e-4 - b1) < 1e-9
    for r in (0.01, 0.1):
        assert abs((ora.density_bias(r + 1e-4, up, o, b1, b2) - ora.density_bias(r, up, o, b1, b2)) / 1e-4 - b2) < 1e-9
    assert ora.density_bias(0.2, up, o, b1, b2) > 0 > ora.density_bias(0.1, up, o, b1, b2)


@pytest.mark.parametrize("ex", GOLD["regularizer_grad"], ids=lambda e: e["cite"][:24])
def test_regularizer_grad_golden(ex):
    """From a zero accumulator with no data gradient, one step stores acc = g^2 with g the
    regulariser gradient 2*lambda*(w + b), and moves w against its sign."""
    w0 = np.array([ex["w"]], np.float32)
    w1, acc = ora.adagrad_step(w0, np.zeros(1, np.float32), np.zeros(1, np.float32), ex["b"], ex["lambda"],
                               0.01, 1e-8)
    assert abs(float(acc[0]) - np.float32(ex["grad"]) ** 2) <= 2e-7 * max(ex["grad"] ** 2, 1e-30)
    if ex["grad"] == 0.0:
        assert acc[0] == 0.0 and w1[0] == w0[0]
    else:
        assert np.sign(w0[0] - w1[0]) == np.sign(ex["grad"])


def test_adagrad_constant_gradient_closed_form():
    """Constant gradient g for T steps: acc_T = T g^2 and w_T = w_0 - lr * sum_t g / (sqrt(t)|g| + eps)
    (the Adagrad recurrence solved in closed form), per weight; zero gradient leaves both alone."""
    rng = np.random.default_rng(7)
    n, T, lr, eps = 64, 40, 0.05, 1e-6
    w0 = rng.uniform(-1, 1, n).astype(np.float32)
    g = rng.uniform(-2, 2, n).astype(np.float32)
    g[:4] = 0.0
    w, acc = w0.copy(), np.zeros(n, np.float32)
    for _ in range(T):
        w, acc = ora.adagrad_step(w, g, acc, 0.0, 0.0, lr, eps)
    gd = g.astype(np.float64)
    t = np.arange(1, T + 1, dtype=np.float64)[:, None]
    w_closed = w0.astype(np.float64) - lr * np.sum(gd[None, :] / (np.sqrt(t) * np.abs(gd)[None, :] + eps), axis=0)
    np.testing.assert_allclose(acc, T * gd * gd, rtol=T * 1.2e-7, atol=0)
    np.testing.assert_allclose(w, w_closed, rtol=0, atol=T * 2e-7)
    assert np.array_equal(w[:4], w0[:4]) and np.all(acc[:4] == 0)


def _run_epochs(values, eps):
    """One weight observed at successive epoch ends; returns the epoch (1-based) it got pruned."""
    keys = np.array([5], np.uint64)
    acc = np.zeros(1, np.float32)
    warn = np.zeros(1, np.uint8)
    for ep, v in enumerate(values, start=1):
        keys, w, acc, warn = ora.prune(keys, np.array([v], np.float32)[: keys.size], acc, warn, eps)
        if keys.size == 0:
            return ep
    return None


@pytest.mark.parametrize("ex", GOLD["prune"], ids=lambda e: e["cite"][:24])
def test_prune_golden(ex):
    assert _run_epochs(ex["epochs"], ex["eps"]) == ex["pruned_after_epoch"]


def test_prune_monotone_and_ordered():
    """Pruning only removes (the count never grows: 'every pruning reduces the number of non-zero
    weights'), keeps key order, and a weight is never removed at its first low observation."""
    rng = np.random.default_rng(3)
    n = 500
    keys = np.sort(rng.choice(10_000, n, replace=False)).astype(np.uint64)
    acc = rng.uniform(0, 1, n).astype(np.float32)
    warn = np.zeros(n, np.uint8)
    first_low = {}
    prev = n
    for ep in range(6):
        w = rng.normal(0, 0.02, keys.size).astype(np.float32)
        for k, v in zip(keys.tolist(), w.tolist()):
            if abs(v) < 0.01:
                first_low.setdefault(k, ep)
        nk, nw, na, nwr = ora.prune(keys, w, acc, warn, 0.01)
        assert nk.size <= prev and np.all(np.diff(nk.astype(np.int64)) > 0)
        assert np.isin(nk, keys).all()
        removed = np.setdiff1d(keys, nk)
        for k in removed.tolist():
            assert first_low[k] < ep
        prev, keys, acc, warn = nk.size, nk, na, nwr


def test_to_dense_pins():
    """sparseToDense (Table 2): every stored entry lands at the cell its decoded index
    (b, c, p) names -- numpy's row-major ravel of the decoded tuple -- and all other cells are 0;
    the dense conv of the bridge equals the bridge of the exact sparse conv (dense xcorr at the
    support, zero elsewhere)."""
    x = uniform_map(2, 3, (5, 6, 7), 0.2, 61)
    d = ora.to_dense(x)
    idx = np.zeros((x.keys.size, 5), np.int64)
    for i, k in enumerate(x.keys.tolist()):
        idx[i] = ora.decode_key(k, x.dims, x.batch, x.channels)
    ref = np.zeros_like(d)
    ref[tuple(idx.T)] = x.values
    np.testing.assert_array_equal(d, ref)
    import torch
    w = sparse_filter(3, 2, (3, 3, 3), 1.0, 62)
    yk, yv, _, _ = ora.conv_fwd(x, w, None)
    yd = ora.to_dense(COO(2, 2, x.dims, yk, yv))
    wd = np.zeros((2, 3, 27), np.float64)
    for k, v in zip(w.keys.tolist(), w.values.tolist()):
        wd[k // (3 * 27), (k // 27) % 3, k % 27] = v
    dense = torch.nn.functional.conv3d(torch.from_numpy(d.astype(np.float64)), torch.from_numpy(wd.reshape(2, 3, 3, 3, 3)),
                                       padding=1).numpy()
    sup = yd != 0
    np.testing.assert_allclose(yd[sup], dense[sup], rtol=1e-6, atol=1e-6)


# ------------------------------------------------------------------ memory model
def _table1():
    with open(os.path.join(os.path.dirname(__file__), "golden", "table1_memory.json")) as f:
        return json.load(f)


def test_memory_estimate_table1():
    """Every cell of Table 1 within one unit of its printed last digit (the paper
    rounds inconsistently: dense 32^3 = 0.0336 GB is printed 0.04, temp 128^3 = 0.0168 as 0.016)."""
    t = _table1()
    for r in (32, 64, 128, 256):
        m64 = ora.memory_estimate(t["ndim"], r, t["batch"], t["channels"], 1.0 / r, 64)
        m32 = ora.memory_estimate(t["ndim"], r, t["batch"], t["channels"], 1.0 / r, 32)
        got = {"dense": m64["dense"], "sparse64": m64["sparse"], "temp": m64["temp"],
               "sparse32": None if m32 is None else m32["sparse"]}
        for row, vals in t["rows"].items():
            want = vals[str(r)]
            if want is None:
                assert got[row] is None, (row, r)
                continue
            unit = t["printed_unit"][row][str(r)]
            assert abs(got[row] / 1e9 - want) <= unit + 1e-12, (row, r, got[row] / 1e9, want)


def test_memory_estimate_paper_statements():
    """P:45 (3x at 100 %, break-even 33 %, 97 % less at 1 %) and P:315 (170x at 512^3)."""
    st = _table1()["statements"]
    full = ora.memory_estimate(3, 64, 1, 1, 1.0, 64)
    assert full["sparse"] / full["dense"] == st["dense_vs_sparse64_at_full_density"]["value"]
    # break-even: sparse == dense at rho = 4 / 12
    be = st["break_even_density"]["value"]
    m = ora.memory_estimate(1, 3 * 2 ** 20, 1, 1, be, 64)
    assert abs(m["sparse"] / m["dense"] - 1.0) < 1e-6
    one = ora.memory_estimate(3, 100, 1, 1, 0.01, 64)
    assert abs((1.0 - one["sparse"] / one["dense"]) - st["saving_at_1pct"]["value"]) < 1e-12
    m512 = ora.memory_estimate(3, 512, 32, 8, 1.0 / 512, 64)
    assert int(m512["dense"] / m512["sparse"]) == st["ratio_at_512"]["value"]
    # 32-bit indices: exactly the cells < 2^32, 8 of 12 bytes per entry
    assert ora.memory_estimate(3, 256, 32, 8, 1 / 256, 32) is None
    assert ora.memory_estimate(3, 256, 32, 7, 1 / 256, 32) is not None
    a, b = ora.memory_estimate(3, 128, 32, 8, 1 / 128, 32), ora.memory_estimate(3, 128, 32, 8, 1 / 128, 64)
    assert a["sparse"] * 12 == b["sparse"] * 8 and a["dense"] == b["dense"] and a["temp"] == b["temp"]

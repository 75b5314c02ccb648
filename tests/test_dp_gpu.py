"""Data-parallel parity on one GPU with virtual shards (SURVEY §4 T3(i), §8(e) "Parity"): the
C4-shaped step (smaller grid) as 2 / 4 / 8 sequential shards through dp.shard_map and the C-ABI.
Per-sample outputs and dx must equal the unsharded call bit for bit; the shards' fp64 dw / dbias
partials (sparse_conv_bwd_f64) summed in fp64 and rounded once (spc_round_f64) must equal the
unsharded dw / dbias bit for bit on dyadic data and to within one fp32 ulp otherwise, and the
oracle's full-batch gradient within the tolerance rule (bit for bit on dyadic data)."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as ora
from synth import uniform_map, sparse_filter, bias_vector, grad_values
from tests._compare import assert_values_close

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

B, C, DIMS, RHO_D, RHO_F = 8, 8, (64, 48, 64), 0.02, 0.5


def _host(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module")
def problem():
    res = {}
    for values in ("dyadic", "continuous"):
        x = uniform_map(B, C, DIMS, RHO_D, 5100, values=values)
        w = sparse_filter(C, C, (3, 3, 3), RHO_F, 5101, values=values)
        bias = bias_vector(C, 5102, values=values)
        V = int(np.prod(DIMS))
        k = V // 20
        yk, yv, _, _ = ora.conv_fwd(x, w, bias, attn=ora.ATTN_MAGNITUDE, k=k)
        dy = grad_values(yk.shape[0], 5103, values=values)
        dx, dw, db, dxa, dwa = ora.conv_bwd(x, w, yk, dy, with_abs=True)
        res[values] = dict(x=x, w=w, bias=bias, k=k, yk=yk, dy=dy, dx=dx, dw=dw, db=db, dwa=dwa, V=V)
    return res


@pytest.mark.parametrize("values", ["dyadic", "continuous"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_virtual_shards_match_unsharded_and_oracle(cuda_lib, problem, values, world):
    spc = cuda_lib
    p = problem[values]
    x, w, bias, k, V = p["x"], p["w"], p["bias"], p["k"], p["V"]
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
    W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
    bt = torch.from_numpy(bias).cuda()
    # unsharded reference run (also through the C-ABI)
    Y = spc.sparse_conv_fwd(X, W, bt, "magnitude", k)
    yk_all, yv_all = (_host(t) for t in Y.trimmed())
    yk_all = yk_all.view(np.uint64)
    if values == "dyadic":   # the forward itself against the oracle
        np.testing.assert_array_equal(yk_all, p["yk"])
    # dy is a function of the kept key set: use the oracle's keys for the backward (the GPU's
    # keys equal them on dyadic data; on continuous data near-threshold swaps are possible)
    Yo = spc.SparseMap.from_arrays(p["yk"], np.zeros(p["yk"].shape[0], np.float32), B, C, DIMS)
    dy_t = torch.from_numpy(p["dy"]).cuda()
    dx_u, dw_u, db_u = spc.sparse_conv_bwd(X, W, Yo, dy_t)
    dx_u, dw_u, db_u = _host(dx_u), _host(dw_u), _host(db_u)

    span_x = np.uint64(C * V)
    dw_acc = torch.zeros(w.nnz, dtype=torch.float64, device="cuda")
    db_acc = torch.zeros(C, dtype=torch.float64, device="cuda")
    for r in range(world):
        b0, b1 = spc.dp.shard_range(B, world, r)
        Xr = spc.dp.shard_map(X, world, r)
        Yr = spc.sparse_conv_fwd(Xr, W, bt, "magnitude", k)
        ykr, yvr = (_host(t) for t in Yr.trimmed())
        lo, hi = np.searchsorted(yk_all, np.uint64(b0) * span_x), np.searchsorted(yk_all, np.uint64(b1) * span_x)
        np.testing.assert_array_equal(ykr.view(np.uint64), yk_all[lo:hi] - np.uint64(b0) * span_x)
        np.testing.assert_array_equal(yvr, yv_all[lo:hi])
        # backward of the shard: dx (fp32) and the fp64 partials of dw / dbias
        lo, hi = np.searchsorted(p["yk"], np.uint64(b0) * span_x), np.searchsorted(p["yk"], np.uint64(b1) * span_x)
        Yor = spc.SparseMap.from_arrays(p["yk"][lo:hi] - np.uint64(b0) * span_x, np.zeros(hi - lo, np.float32),
                                        b1 - b0, C, DIMS)
        plan = spc.BwdPlan(Xr, W, Yor)
        dxr = torch.empty(max(Xr.nnz_bound, 1), device="cuda")
        ar = spc.dp.GradAllReduce(w.nnz, C, "cuda")
        plan.f64(Xr, W, Yor, dy_t[lo:hi].contiguous(), dxr, ar.dw64, ar.db64)
        dw_acc += ar.dw64                      # the all-reduce SUM of virtual rank r
        db_acc += ar.db64
        xlo, xhi = np.searchsorted(x.keys, np.uint64(b0) * span_x), np.searchsorted(x.keys, np.uint64(b1) * span_x)
        np.testing.assert_array_equal(_host(dxr)[:xhi - xlo], dx_u[xlo:xhi])
    dw_s = _host(spc.round_f64(dw_acc, torch.empty(w.nnz, device="cuda")))
    db_s = _host(spc.round_f64(db_acc, torch.empty(C, device="cuda")))
    if values == "dyadic":   # every fp64 sum exact: identical bits everywhere
        np.testing.assert_array_equal(dw_s, dw_u)
        np.testing.assert_array_equal(db_s, db_u)
        np.testing.assert_array_equal(dw_s, p["dw"])
        np.testing.assert_array_equal(db_s, p["db"])
    else:
        assert np.all(np.abs(dw_s - dw_u) <= np.spacing(np.abs(dw_u)))
        assert np.all(np.abs(db_s - db_u) <= np.spacing(np.abs(db_u)))
        assert_values_close(dw_s, p["dw"], p["dwa"], "sharded dw")
        assert_values_close(db_s, p["db"], np.full(C, np.abs(p["dy"]).sum()), "sharded dbias")


def test_shard_map_partitions_device_map(cuda_lib):
    spc = cuda_lib
    x = uniform_map(7, 3, (9, 10, 11), 0.1, 5200)
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
    for world in (1, 2, 3, 7):
        parts = [spc.dp.shard_map(X, world, r) for r in range(world)]
        assert sum(pm.batch for pm in parts) == 7
        keys = []
        for r, pm in enumerate(parts):
            b0, _ = spc.dp.shard_range(7, world, r)
            keys.append(_host(pm.keys).view(np.uint64) + np.uint64(b0 * 3 * 990))
        np.testing.assert_array_equal(np.concatenate(keys), x.keys)

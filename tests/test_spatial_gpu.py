"""Spatial sharding of a sample's grid on one GPU with virtual shards
(spatial.LoopbackComm: every rank in this process, lockstep): the first spatial dimension is cut
into 2..4 plane ranges, each rank convolves its planes plus halo planes received from its
neighbours, attention is selected over the whole (b, oc) segment by the distributed radix select,
and the backward returns the halo inputs' dx partials to their owners.

On dyadic data (every sum exact) each rank's output keys / values, dx, and the all-reduced dw /
dbias must equal the single-GPU layer bit for bit -- and the oracle (Alg. 1 / Alg. 2, P:54-84,
P:137-161) on the full grid. Continuous data: the same keys (the kept set of every segment) and
values within the tolerance rule."""
from __future__ import annotations

import numpy as np
import pytest

import oracle as ora
from synth import uniform_map, sparse_filter, bias_vector, grad_values

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ORA_ATTN = {"none": None, "magnitude": "ATTN_MAGNITUDE", "raw": "ATTN_RAW"}

CASES = [
    # (batch, c_in, c_out, dims, ksize, rho_d, rho_f, world)
    (2, 3, 4, (12, 10, 14), (3, 3, 3), 0.08, 0.5, 2),
    (2, 3, 4, (12, 10, 14), (3, 3, 3), 0.08, 0.5, 4),
    (1, 2, 3, (7, 9, 11), (5, 3, 3), 0.15, 0.6, 3),     # halo of 2 planes, shards of 3/2/2
    (2, 2, 2, (16, 40), (3, 5), 0.1, 0.7, 3),           # 2D
    (1, 2, 2, (6, 5, 4, 7), (3, 3, 3, 3), 0.1, 0.4, 2), # rank 4
    (1, 4, 4, (9, 8, 8), (1, 3, 3), 0.1, 0.5, 3),       # no halo along the planes
]


def _host(t):
    return t.detach().cpu().numpy()


def _run(case, attn, values, seed):
    import paper_1801_10585_b200 as spc
    from paper_1801_10585_b200.spatial import LoopbackComm, SpatialConv, extract_planes

    b, ci, co, dims, ks, rd, rf, world = case
    x = uniform_map(b, ci, dims, rd, seed, values=values)
    w = sparse_filter(ci, co, ks, rf, seed + 1, values=values)
    bias = bias_vector(co, seed + 2, values=values)
    V = int(np.prod(dims))
    k = max(1, V // 6) if attn != "none" else 0
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
    W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
    bt = torch.from_numpy(bias).cuda()
    Y = spc.sparse_conv_fwd(X, W, bt, attn, k).exact()
    comm = LoopbackComm(world)
    layer = SpatialConv(comm, dims[0])
    rng = layer.ranges()
    xs = [extract_planes(X, a, e)[0].exact() for a, e in rng]
    ys = layer.forward(xs, W, bt, attn, k)
    ys = [y.exact() for y in ys]
    dy = torch.from_numpy(grad_values(Y.nnz_bound, seed + 3, values=values)).cuda()
    dX, dW, dB = spc.sparse_conv_bwd(X, W, Y, dy)
    dys, refs, xidx = [], [], []
    for (a, e) in rng:
        ry, yi = extract_planes(Y, a, e, src_index=True)
        ry = ry.exact()
        refs.append(ry)
        dys.append(dy[yi[:ry.nnz_bound]].contiguous())
        _, xi = extract_planes(X, a, e, src_index=True)
        xidx.append(xi)
    outs = layer.backward(xs, W, ys, dys)
    return dict(x=x, w=w, bias=bias, k=k, Y=Y, ys=ys, refs=refs, dy=dy, dX=dX, dW=dW, dB=dB, outs=outs,
                xs=xs, xidx=xidx, V=V)


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{len(c[3])}d-{c[3]}-k{c[4][0]}-w{c[7]}")
@pytest.mark.parametrize("attn", ["magnitude", "raw", "none"])
def test_spatial_shards_bit_exact_dyadic(cuda_lib, case, attn):
    r = _run(case, attn, "dyadic", 7300 + len(case[3]))
    # the unsharded layer against the oracle on the whole grid (Alg. 1 with attention)
    a = getattr(ora, ORA_ATTN[attn]) if ORA_ATTN[attn] else ora.ATTN_NONE
    ok, ov, _, _ = ora.conv_fwd(r["x"], r["w"], r["bias"], attn=a, k=r["k"])
    assert np.array_equal(_host(r["Y"].keys).view(np.uint64), ok)
    assert np.array_equal(_host(r["Y"].values), ov)
    for j, (y, ref) in enumerate(zip(r["ys"], r["refs"])):
        assert y.nnz_bound == ref.nnz_bound, f"rank {j}: {y.nnz_bound} kept vs {ref.nnz_bound}"
        assert torch.equal(y.keys, ref.keys), f"rank {j}: output keys differ"
        assert torch.equal(y.values, ref.values), f"rank {j}: output values differ"
    odx, odw, odb, _, _ = ora.conv_bwd(r["x"], r["w"], ok, _host(r["dy"]))
    for j, ((dx, dw, db), xi, xsh) in enumerate(zip(r["outs"], r["xidx"], r["xs"])):
        ref_dx = r["dX"][xi[:xsh.nnz_bound]]
        assert torch.equal(dx, ref_dx), f"rank {j}: dx differs"
        assert np.array_equal(_host(dw), odw), f"rank {j}: dw differs from the oracle"
        assert np.array_equal(_host(db), odb), f"rank {j}: dbias differs from the oracle"
    assert np.array_equal(_host(r["dX"]), odx)


@pytest.mark.parametrize("case", CASES[:3], ids=lambda c: f"{c[3]}-w{c[7]}")
def test_spatial_shards_continuous(cuda_lib, case):
    r = _run(case, "magnitude", "continuous", 7400)
    for j, (y, ref) in enumerate(zip(r["ys"], r["refs"])):
        assert torch.equal(y.keys, ref.keys), f"rank {j}: kept set differs"
        torch.testing.assert_close(y.values, ref.values, rtol=1e-5, atol=1e-6)
    for j, ((dx, dw, db), xi, xsh) in enumerate(zip(r["outs"], r["xidx"], r["xs"])):
        torch.testing.assert_close(dx, r["dX"][xi[:xsh.nnz_bound]], rtol=1e-5, atol=1e-5)
        torch.testing.assert_close(dw, r["dW"], rtol=1e-5, atol=1e-5)
        torch.testing.assert_close(db, r["dB"], rtol=1e-5, atol=1e-5)


def test_spatial_select_ties_and_small_segments(cuda_lib):
    """Binary values (massive score ties, R7: ties to the smaller global position) and k larger
    than some segments' support (keep all)."""
    import paper_1801_10585_b200 as spc
    from paper_1801_10585_b200.spatial import LoopbackComm, SpatialConv, extract_planes

    dims = (10, 8, 8)
    x = uniform_map(2, 2, dims, 0.05, 7500, values="dyadic")
    x.values[:] = 1.0
    w = sparse_filter(2, 3, (3, 3, 3), 0.5, 7501, values="dyadic")
    w.values[:] = 0.5
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
    W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
    for k in (7, 40, 10 ** 6):
        Y = spc.sparse_conv_fwd(X, W, None, "magnitude", k).exact()
        layer = SpatialConv(LoopbackComm(3), dims[0])
        xs = [extract_planes(X, a, e)[0].exact() for a, e in layer.ranges()]
        ys = layer.forward(xs, W, None, "magnitude", k)
        for (a, e), y in zip(layer.ranges(), ys):
            ref = extract_planes(Y, a, e)[0].exact()
            y = y.exact()
            assert torch.equal(y.keys, ref.keys) and torch.equal(y.values, ref.values), k


def test_spatial_empty_shard_and_thin_shard_error(cuda_lib):
    import paper_1801_10585_b200 as spc
    from paper_1801_10585_b200.spatial import LoopbackComm, SpatialConv, extract_planes

    dims = (8, 6, 6)
    x = uniform_map(1, 2, dims, 0.05, 7600, values="dyadic")
    keep = (x.keys % np.uint64(np.prod(dims))) < np.uint64(4 * 36)   # inputs only in planes 0..3
    X = spc.SparseMap.from_arrays(x.keys[keep], x.values[keep], 1, 2, dims)
    w = sparse_filter(2, 2, (3, 3, 3), 0.6, 7601, values="dyadic")
    W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
    Y = spc.sparse_conv_fwd(X, W, None, "magnitude", 20).exact()
    layer = SpatialConv(LoopbackComm(4), dims[0])
    xs = [extract_planes(X, a, e)[0].exact() for a, e in layer.ranges()]
    assert xs[3].nnz_bound == 0
    ys = layer.forward(xs, W, None, "magnitude", 20)
    for (a, e), y in zip(layer.ranges(), ys):
        ref = extract_planes(Y, a, e)[0].exact()
        y = y.exact()
        assert torch.equal(y.keys, ref.keys) and torch.equal(y.values, ref.values)
    w5 = sparse_filter(2, 2, (5, 3, 3), 0.6, 7602, values="dyadic")
    W5 = spc.SparseFilter.from_arrays(w5.keys, w5.values, w5.c_in, w5.c_out, w5.ksize)
    thin = SpatialConv(LoopbackComm(8), dims[0])   # one plane per rank < halo of 2
    with pytest.raises(ValueError):
        thin.forward([extract_planes(X, a, e)[0].exact() for a, e in thin.ranges()], W5, None, "magnitude", 20)


def _dist_worker(rank, world, port, q):
    """One spatial rank per process (gloo with host staging; the kernels of each process run
    independently on the one GPU): DistComm's real halo exchange and all-reduces."""
    import os

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1801_10585_b200 as spc
        from paper_1801_10585_b200.spatial import DistComm, SpatialConv, extract_planes

        torch.cuda.set_device(0)
        spc.load()
        dims = (12, 10, 14)
        x = uniform_map(2, 3, dims, 0.08, 7700, values="dyadic")
        w = sparse_filter(3, 4, (3, 3, 3), 0.5, 7701, values="dyadic")
        bias = bias_vector(4, 7702, values="dyadic")
        X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
        W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
        bt = torch.from_numpy(bias).cuda()
        k = 250
        Y = spc.sparse_conv_fwd(X, W, bt, "magnitude", k).exact()
        dy = torch.from_numpy(grad_values(Y.nnz_bound, 7703, values="dyadic")).cuda()
        dX, dW, dB = spc.sparse_conv_bwd(X, W, Y, dy)
        layer = SpatialConv(DistComm(), dims[0])
        (a, e), = layer.ranges()
        xr = extract_planes(X, a, e)[0].exact()
        [y] = layer.forward([xr], W, bt, "magnitude", k)
        y = y.exact()
        ref, yi = extract_planes(Y, a, e, src_index=True)
        ref = ref.exact()
        [(dx, dw, db)] = layer.backward([xr], W, [y], [dy[yi[:ref.nnz_bound]].contiguous()])
        _, xi = extract_planes(X, a, e, src_index=True)
        ok = (torch.equal(y.keys, ref.keys) and torch.equal(y.values, ref.values)
              and torch.equal(dx, dX[xi[:xr.nnz_bound]]) and torch.equal(dw, dW) and torch.equal(db, dB))
        q.put((rank, bool(ok), int(y.nnz_bound)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_spatial_distcomm_processes(cuda_lib, world):
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_dist_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in got), got

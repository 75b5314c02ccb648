"""Multi-process (world_size 2, gloo, CPU) coverage of the data-parallel path: batch sharding
by per-sample seeds and the SUM all-reduce of the fp64 partials dw64||db64 with one final
rounding (reading R13; dp.GradAllReduce). The oracle stands in for the per-rank compute
(ora.conv_bwd64 = Alg. 2 with the fp64 sums before rounding), so the sharded result must equal
the full-batch oracle gradient -- bit for bit on dyadic data (every fp64 sum exact)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1801_10585_b200.dp import GradAllReduce, shard_range, max_over_ranks, sum_over_ranks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(values="continuous"):
    import oracle as ora
    from synth import uniform_map, sparse_filter, bias_vector

    B, dims = 6, (10, 9, 8)
    w = sparse_filter(2, 3, (3, 3, 3), 0.5, 5, values=values)
    bias = bias_vector(3, 5, values=values)
    return ora, uniform_map, B, dims, w, bias


def _dy(n, b0, values):
    rng = np.random.default_rng(1000 + b0)
    if values == "dyadic":
        return (rng.integers(-64, 65, n) / 64.0).astype(np.float32)
    return rng.uniform(-1, 1, n).astype(np.float32)


def _worker(rank, world, port, out, values):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ora, uniform_map, B, dims, w, bias = _setup(values)
    b0, b1 = shard_range(B, world, rank)
    x = uniform_map(b1 - b0, 2, dims, 0.1, 77, b0=b0, values=values)        # this rank's shard only
    V = int(np.prod(dims))
    yk, _, _, _ = ora.conv_fwd(x, w, bias, attn=ora.ATTN_MAGNITUDE, k=V // 10)
    dy = _dy(yk.shape[0], b0, values)
    _, dw64, db64, _, _ = ora.conv_bwd64(x, w, yk, dy)
    ar = GradAllReduce(dw64.shape[0], db64.shape[0], "cpu")
    ar.dw64.copy_(torch.from_numpy(dw64))
    ar.db64.copy_(torch.from_numpy(db64))
    dw_t, db_t = torch.empty(dw64.shape[0]), torch.empty(db64.shape[0])
    ar(dw_t, db_t)
    t = max_over_ranks(float(rank + 1), "cpu")
    s = sum_over_ranks([1.0, float(x.nnz)], "cpu")
    out[rank] = (dw_t.numpy().copy(), db_t.numpy().copy(), x.keys.copy(), t, s)
    dist.destroy_process_group()


def test_shard_range_partitions_batch():
    for B in (1, 7, 64):
        for world in (1, 2, 3, 8):
            rs = [shard_range(B, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == B
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("values", ["continuous", "dyadic"])
def test_gloo_world2_sharded_grads_equal_full_batch(values):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, out, values), nprocs=world, join=True, start_method="spawn")
    ora, uniform_map, B, dims, w, bias = _setup(values)
    x = uniform_map(B, 2, dims, 0.1, 77, values=values)
    V = int(np.prod(dims))
    yk, _, _, _ = ora.conv_fwd(x, w, bias, attn=ora.ATTN_MAGNITUDE, k=V // 10)
    # dy drawn per shard in the workers: rebuild the same full-batch dy
    span = np.uint64(3 * V)
    dys = []
    for r in range(world):
        b0, b1 = shard_range(B, world, r)
        lo, hi = np.searchsorted(yk, np.uint64(b0) * span), np.searchsorted(yk, np.uint64(b1) * span)
        dys.append(_dy(hi - lo, b0, values))
    dy = np.concatenate(dys)
    _, dw, db, _, dwa = ora.conv_bwd(x, w, yk, dy, with_abs=True)
    for r in range(world):
        gdw, gdb, keys, t, s = out[r]
        if values == "dyadic":   # every fp64 partial and sum exact: one rounding, identical bits
            np.testing.assert_array_equal(gdw, dw)
            np.testing.assert_array_equal(gdb, db)
        else:                    # fp64 sums in another order, rounded once: at most 1 ulp apart
            assert np.all(np.abs(gdw - dw) <= np.spacing(np.abs(dw)))
            assert np.all(np.abs(gdb - db) <= np.spacing(np.abs(db)))
        assert t == 2.0 and s[0] == 2.0
    # shards generated from per-sample seeds are exactly the rows of the full batch
    k0 = out[0][2]
    k1 = out[1][2]
    b0, b1 = shard_range(B, world, 1)
    full0 = x.keys[x.keys < np.uint64(b0) * np.uint64(2 * V)]
    np.testing.assert_array_equal(k0, full0)
    full1 = x.keys[x.keys >= np.uint64(b0) * np.uint64(2 * V)] - np.uint64(b0) * np.uint64(2 * V)
    np.testing.assert_array_equal(k1, full1)

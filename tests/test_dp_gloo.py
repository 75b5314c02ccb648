"""Multi-process (world_size 2, gloo, CPU) coverage of the data-parallel path: batch sharding
by per-sample seeds and the SUM all-reduce of dw||dbias (reading R13). The oracle stands in for
the per-rank compute, so the sharded result must equal the full-batch oracle gradient."""
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


def _setup():
    import oracle as ora
    from synth import uniform_map, sparse_filter, bias_vector

    B, dims = 6, (10, 9, 8)
    w = sparse_filter(2, 3, (3, 3, 3), 0.5, 5, values="continuous")
    bias = bias_vector(3, 5)
    return ora, uniform_map, B, dims, w, bias


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ora, uniform_map, B, dims, w, bias = _setup()
    b0, b1 = shard_range(B, world, rank)
    x = uniform_map(b1 - b0, 2, dims, 0.1, 77, b0=b0)        # this rank's shard only
    V = int(np.prod(dims))
    yk, _, _, _ = ora.conv_fwd(x, w, bias, attn=ora.ATTN_MAGNITUDE, k=V // 10)
    rng = np.random.default_rng(1000 + b0)
    dy = rng.uniform(-1, 1, yk.shape[0]).astype(np.float32)
    _, dw, db, _, _ = ora.conv_bwd(x, w, yk, dy)
    dw_t, db_t = torch.from_numpy(dw.copy()), torch.from_numpy(db.copy())
    GradAllReduce(dw.shape[0], db.shape[0], "cpu")(dw_t, db_t)
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


def test_gloo_world2_sharded_grads_equal_full_batch():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, join=True, start_method="spawn")
    ora, uniform_map, B, dims, w, bias = _setup()
    x = uniform_map(B, 2, dims, 0.1, 77)
    V = int(np.prod(dims))
    yk, _, _, _ = ora.conv_fwd(x, w, bias, attn=ora.ATTN_MAGNITUDE, k=V // 10)
    # dy drawn per shard in the workers: rebuild the same full-batch dy
    span = np.uint64(3 * V)
    dys = []
    for r in range(world):
        b0, b1 = shard_range(B, world, r)
        lo, hi = np.searchsorted(yk, np.uint64(b0) * span), np.searchsorted(yk, np.uint64(b1) * span)
        dys.append(np.random.default_rng(1000 + b0).uniform(-1, 1, hi - lo).astype(np.float32))
    dy = np.concatenate(dys)
    _, dw, db, _, dwa = ora.conv_bwd(x, w, yk, dy, with_abs=True)
    for r in range(world):
        gdw, gdb, keys, t, s = out[r]
        # per-rank fp32 partials summed in fp64, rounded once: within a few fp32 ulps
        assert np.all(np.abs(gdw - dw) <= 1e-6 * dwa + 1e-5 * np.abs(dw))
        np.testing.assert_allclose(gdb, db, rtol=1e-5, atol=1e-6)
        assert t == 2.0 and s[0] == 2.0
    # shards generated from per-sample seeds are exactly the rows of the full batch
    k0 = out[0][2]
    k1 = out[1][2]
    b0, b1 = shard_range(B, world, 1)
    full0 = x.keys[x.keys < np.uint64(b0) * np.uint64(2 * V)]
    np.testing.assert_array_equal(k0, full0)
    full1 = x.keys[x.keys >= np.uint64(b0) * np.uint64(2 * V)] - np.uint64(b0) * np.uint64(2 * V)
    np.testing.assert_array_equal(k1, full1)

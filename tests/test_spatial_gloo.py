"""Host logic of the spatial sharding on CPU: the plane partition and the
two collectives of spatial.DistComm -- the neighbour halo exchange (sizes first, then payloads;
point-to-point) and the SUM all-reduce -- under gloo with world sizes 2 and 3, checked against
LoopbackComm (all ranks in one process), which the GPU parity tests drive."""
from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1801_10585_b200.spatial import DistComm, LoopbackComm, plane_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_plane_range_partitions():
    for planes in (1, 5, 7, 64, 129):
        for world in (1, 2, 3, 4, 8):
            rs = [plane_range(planes, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == planes
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [e - a for a, e in rs]
            assert max(sizes) - min(sizes) <= 1


def _payload(r, side):
    """Deterministic variable-size payload rank r sends to its left (side 0) / right (1) neighbour;
    rank 1 sends nothing to the left (empty halo)."""
    n = 0 if (r == 1 and side == 0) else 3 + 2 * r + side
    keys = torch.arange(n, dtype=torch.int64) + 1000 * r + 100 * side
    vals = torch.arange(n, dtype=torch.float32) * 0.5 + r
    return [keys, vals]


def _expected(world):
    to_left = [_payload(r, 0) if r > 0 else None for r in range(world)]
    to_right = [_payload(r, 1) if r < world - 1 else None for r in range(world)]
    return LoopbackComm(world).exchange(to_left, to_right)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = DistComm()
        tl = _payload(rank, 0) if rank > 0 else None
        tr = _payload(rank, 1) if rank < world - 1 else None
        fl, fr = comm.exchange([tl], [tr])
        t = torch.arange(6, dtype=torch.int32) * (rank + 1)
        comm.allreduce_sum([t])
        q.put((rank, [None if fl[0] is None else [x.tolist() for x in fl[0]]],
               [None if fr[0] is None else [x.tolist() for x in fr[0]]], t.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distcomm_exchange_and_allreduce_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, fl, fr, t = q.get(timeout=120)
        got[rank] = (fl[0], fr[0], t)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    efl, efr = _expected(world)
    tot = sum(r + 1 for r in range(world))
    for r in range(world):
        fl, fr, t = got[r]
        assert (fl is None) == (efl[r] is None) and (fr is None) == (efr[r] is None)
        if fl is not None:
            assert fl == [x.tolist() for x in efl[r]]
        if fr is not None:
            assert fr == [x.tolist() for x in efr[r]]
        assert t == [i * tot for i in range(6)]

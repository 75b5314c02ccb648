"""Data-parallel plumbing (north star: "Work is partitioned across the 8 B200s of one box by
sharding the batch, with an NCCL all-reduce over NVLink used only for the weight gradients").

Samples are independent in the forward pass, in dx, in attention, ReLU and pooling; only the
weight and bias gradients are sums over the batch (Alg. 2 accumulates bp_filter over b).
A rank therefore owns a contiguous range of samples (with batch-major keys that is one contiguous
key range of every map, `shard_map`) and the only exchange is one SUM all-reduce of dw||dbias per
layer (reading R13: SUM, not mean, so the sharded gradient equals the full-batch gradient).

The exchanged values are the UNROUNDED fp64 accumulators of each rank's shard
(`BwdPlan.f64` = sparse_conv_bwd_f64); the reduced sum is rounded to fp32 once (spc_round_f64),
so a sharded step reproduces the single-GPU dw bit for bit whenever the fp64 sums are exact.
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.distributed as dist


def shard_range(batch: int, world: int, rank: int) -> Tuple[int, int]:
    """[b0, b1) of the samples rank `rank` owns (contiguous, sizes differ by at most one)."""
    base, rem = divmod(batch, world)
    b0 = rank * base + min(rank, rem)
    return b0, b0 + base + (1 if rank < rem else 0)


def shard_map(x, world: int, rank: int):
    """Rank `rank`'s share of a device SparseMap: its samples' entries (one contiguous key range,
    found by two binary searches on the device keys) re-based to sample 0. Plumbing only (the
    keys are copied, nothing is computed on them but the batch offset)."""
    from .ops import SparseMap

    b0, b1 = shard_range(x.batch, world, rank)
    span = x.channels * x.volume
    n = x.nnz()
    keys = x.keys[:n]
    bounds = torch.tensor([b0 * span, b1 * span], dtype=torch.int64, device=keys.device)
    lo, hi = torch.searchsorted(keys, bounds).tolist()
    k = (keys[lo:hi] - b0 * span).contiguous()
    v = x.values[lo:hi].contiguous()
    return SparseMap(k, v, b1 - b0, x.channels, x.dims, int(k.numel()), None)


class GradAllReduce:
    """SUM over ranks of the fp64 partials dw64 || db64 of one layer (NCCL over NVLink on a GPU
    box, gloo in the CPU tests), then one rounding to fp32 (spc_round_f64).

    `start()` enqueues the all-reduce -- on `stream` when given, after the compute stream's work,
    so that what the caller enqueues next on the compute stream (the next layer's backward, the
    next step's forward) overlaps it; `finish(dw, dbias)` makes the compute stream wait for it and
    rounds. `__call__` = start + finish. Buffers: `dw64`, `db64` (views of one flat fp64 buffer,
    the output arrays of BwdPlan.f64)."""

    def __init__(self, n_w: int, c_out: int, device, group=None, stream: Optional[torch.cuda.Stream] = None):
        self.n_w, self.c_out = int(n_w), int(c_out)
        self.buf = torch.zeros(self.n_w + self.c_out, dtype=torch.float64, device=device)
        self.dw64 = self.buf[:self.n_w]
        self.db64 = self.buf[self.n_w:]
        self.group = group
        self.stream = stream
        self._pending = False

    def _distributed(self) -> bool:
        return dist.is_initialized() and dist.get_world_size(self.group) > 1

    def start(self):
        if not self._distributed():
            return
        if self.stream is not None and self.buf.is_cuda:
            self.stream.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(self.stream):
                dist.all_reduce(self.buf, op=dist.ReduceOp.SUM, group=self.group)
            self._pending = True
        else:
            dist.all_reduce(self.buf, op=dist.ReduceOp.SUM, group=self.group)

    def finish(self, dw: torch.Tensor, dbias: Optional[torch.Tensor] = None):
        if self._pending:
            torch.cuda.current_stream().wait_stream(self.stream)
            self._pending = False
        if self.buf.is_cuda:
            from .ops import round_f64

            round_f64(self.dw64, dw[:self.n_w])
            if dbias is not None:
                round_f64(self.db64, dbias[:self.c_out])
        else:   # CPU (gloo) tests: the same single rounding
            dw[:self.n_w].copy_(self.dw64.to(torch.float32))
            if dbias is not None:
                dbias[:self.c_out].copy_(self.db64.to(torch.float32))
        return dw, dbias

    def __call__(self, dw: torch.Tensor, dbias: Optional[torch.Tensor] = None):
        self.start()
        return self.finish(dw, dbias)


def max_over_ranks(value: float, device, group=None) -> float:
    """Time-like reductions: the slowest rank defines the step."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(values, device, group=None):
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [float(v) for v in values]
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return [float(v) for v in t.tolist()]

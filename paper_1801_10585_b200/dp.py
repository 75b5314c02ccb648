"""Data-parallel plumbing (north star: "Work is partitioned across the 8 B200s of one box by
sharding the batch, with an NCCL all-reduce over NVLink used only for the weight gradients").

Samples are independent in the forward pass, in dx, in attention, ReLU and pooling; only the
weight and bias gradients are sums over the batch (Alg. 2). A rank therefore owns a
contiguous range of samples (with batch-major keys that is one contiguous key range of every
map) and the only exchange is one SUM all-reduce of dw||dbias per layer (reading R13: SUM,
not mean, so the sharded gradient equals the full-batch gradient). The reduction runs in fp64.
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


class GradAllReduce:
    """Packs dw||dbias into one fp64 buffer and all-reduces it (SUM) on `group`; optionally on a
    side stream so that it overlaps with work queued after it on the compute stream."""

    def __init__(self, n_w: int, c_out: int, device, group=None, stream: Optional[torch.cuda.Stream] = None):
        self.n_w, self.c_out = int(n_w), int(c_out)
        self.buf = torch.empty(self.n_w + self.c_out, dtype=torch.float64, device=device)
        self.group = group
        self.stream = stream

    def __call__(self, dw: torch.Tensor, dbias: torch.Tensor):
        if not dist.is_initialized() or dist.get_world_size(self.group) == 1:
            return dw, dbias
        self.buf[:self.n_w].copy_(dw)
        self.buf[self.n_w:].copy_(dbias)
        if self.stream is not None:
            self.stream.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(self.stream):
                dist.all_reduce(self.buf, op=dist.ReduceOp.SUM, group=self.group)
            torch.cuda.current_stream().wait_stream(self.stream)
        else:
            dist.all_reduce(self.buf, op=dist.ReduceOp.SUM, group=self.group)
        dw.copy_(self.buf[:self.n_w])
        dbias.copy_(self.buf[self.n_w:])
        return dw, dbias


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

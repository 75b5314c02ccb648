"""Spatial sharding of one sample's grid across ranks (beyond the paper,
which holds a whole (b, oc) grid in one GPU's dense temporary buffer).

The first spatial dimension ("planes", the most significant one in the key, reading R11) is cut
into contiguous ranges, rank r owning planes [a_r, e_r) (`plane_range`). A shard map is an
ordinary SparseMap over dims (e_r - a_r, dims[1:]). By Eq. (1) an output depends only on the
inputs within the filter's extent, so rank r computes its outputs exactly from its inputs plus
h = ksize[0] // 2 halo planes from each neighbour. One layer (Alg. 1 forward, Alg. 2 backward):

forward   1. halo exchange: the first / last h planes go to rank r-1 / r+1 (point-to-point);
          2. extended input = [left halo | own planes | right halo] per (b, c) (spc_slab_gather);
          3. the convolution without attention on the extended grid (the library's forward);
          4. the owned planes of its output (spc_slab_gather): the exact response and structural
             support of every owned voxel (halo-plane outputs miss contributions and are dropped);
          5. attention over the whole (b, oc) segment, which no rank holds: an exact
             8-round radix select on the R7 composite with GLOBAL positions (spc_topk_digit_hist,
             one SUM all-reduce of nseg x 256 counts per round, spc_topk_digit_pick), then
             spc_topk_keep_ge -- the same kept set and values as the single-GPU layer.
backward  6. dx, fp64 dw / dbias partials on the extended input against the OWNED kept outputs
             only, so every (input, output) pair of Alg. 2 is counted by exactly one rank;
          7. the halo inputs' dx partials go back to their owners (point-to-point) and are added
             there (spc_index_add); dw || dbias: one SUM all-reduce of the fp64 partials, rounded
             once (as in dp.py).

Communication goes through a `Comm`: `DistComm` (torch.distributed, one rank per process: NCCL
over NVLink on a GPU box, gloo in the CPU tests) or `LoopbackComm` (all ranks in this process,
run in lockstep: virtual shards on one GPU for the parity tests). Every step of the layer runs
in libspconv kernels; this module marshals arguments and moves buffers.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist

from ._lib import ATTN, SlabSrcT, check, load
from .ops import BwdPlan, SparseFilter, SparseMap, _out, _ptr, _stream, _workspace, round_f64, sparse_conv_fwd, \
    sparse_scatter_grad


def plane_range(planes: int, world: int, rank: int) -> Tuple[int, int]:
    """[a, e) of the planes rank `rank` owns (contiguous, sizes differ by at most one)."""
    base, rem = divmod(planes, world)
    a = rank * base + min(rank, rem)
    return a, a + base + (1 if rank < rem else 0)


# ------------------------------------------------------------------ C-ABI marshalling
def slab_gather(sources: Sequence[Tuple[SparseMap, int, int, int]], planes_out: int, src_index: bool = False,
                stream=None) -> Tuple[SparseMap, Optional[torch.Tensor], List[int]]:
    """spc_slab_gather: per (b, c), the concatenation of each source's planes [lo, hi) moved to
    plane + shift of a grid with `planes_out` planes. sources = [(map, lo, hi, shift), ...].
    Returns (map, source index or None, bases of the sources in the index space)."""
    lib = load()
    m0 = sources[0][0]
    nseg = m0.batch * m0.channels
    plane = 1
    for d in m0.dims[1:]:
        plane *= int(d)
    arr = (SlabSrcT * len(sources))()
    bases, bound = [], 0
    for j, (m, lo, hi, shift) in enumerate(sources):
        assert m.batch == m0.batch and m.channels == m0.channels and tuple(m.dims[1:]) == tuple(m0.dims[1:])
        assert m.key_bits == 64, "spatial sharding takes 64-bit keys"
        s = arr[j]
        s.keys = m.keys.data_ptr() if m.keys.numel() else None
        s.values = m.values.data_ptr() if m.values.numel() else None
        s.nnz_dev = None if m.nnz_dev is None else m.nnz_dev.data_ptr()
        s.n, s.planes, s.lo, s.hi, s.shift = int(m.nnz_bound), int(m.dims[0]), int(lo), int(hi), int(shift)
        bases.append(bound)
        bound += int(m.nnz_bound)
    dev = m0.values.device
    ws = C.c_size_t()
    check("spc_slab_gather_query", lib.spc_slab_gather_query(nseg, len(sources), C.byref(ws)))
    w = _workspace(ws.value, dev)
    keys, vals, nnz, o = _out(bound, dev)
    idx = torch.empty(max(bound, 1), dtype=torch.int64, device=dev) if src_index else None
    check("spc_slab_gather", lib.spc_slab_gather(arr, len(sources), nseg, plane, int(planes_out), C.byref(o),
                                                 _ptr(idx), _ptr(w), w.numel(), _stream(stream)))
    dims = (int(planes_out),) + tuple(m0.dims[1:])
    return SparseMap(keys, vals, m0.batch, m0.channels, dims, bound, nnz), idx, bases


def extract_planes(x: SparseMap, a: int, e: int, src_index: bool = False, stream=None):
    """Planes [a, e) of x as a map over (e - a) planes (keys re-based)."""
    y, idx, _ = slab_gather([(x, a, e, -a)], e - a, src_index, stream)
    return y, idx


def place_planes(x: SparseMap, a: int, planes: int, stream=None) -> SparseMap:
    """A shard map (its planes starting at global plane a) as a map over `planes` planes."""
    return slab_gather([(x, 0, x.dims[0], a)], planes, False, stream)[0]


def index_add(idx: torch.Tensor, v: torch.Tensor, out: torch.Tensor, n: Optional[int] = None, stream=None):
    """out[idx[t]] += v[t] (spc_index_add; idx injective)."""
    n = int(v.numel()) if n is None else int(n)
    check("spc_index_add", load().spc_index_add(_ptr(idx), _ptr(v), n, None, _ptr(out), _stream(stream)))
    return out


@dataclass
class _Select:
    prefix: torch.Tensor   # int64 bit patterns of the uint64 prefixes [nseg]
    need: torch.Tensor     # int64 [nseg]
    hist: torch.Tensor     # int32 [nseg * 256]


def _select_init(nseg: int, k: int, dev) -> _Select:
    return _Select(torch.zeros(max(nseg, 1), dtype=torch.int64, device=dev),
                   torch.full((max(nseg, 1),), int(k), dtype=torch.int64, device=dev),
                   torch.zeros(max(nseg, 1) * 256, dtype=torch.int32, device=dev))


def _digit_hist(y: SparseMap, attn: str, p_base: int, st: _Select, shift: int, stream=None):
    st.hist.zero_()
    ys = y.c_struct()
    check("spc_topk_digit_hist", load().spc_topk_digit_hist(C.byref(ys), ATTN[attn], int(p_base), _ptr(st.prefix),
                                                            _ptr(st.need), int(shift), _ptr(st.hist),
                                                            _stream(stream)))


def _digit_pick(nseg: int, st: _Select, shift: int, stream=None):
    check("spc_topk_digit_pick", load().spc_topk_digit_pick(int(nseg), _ptr(st.hist), int(shift), _ptr(st.prefix),
                                                            _ptr(st.need), _stream(stream)))


def keep_ge(y: SparseMap, attn: str, p_base: int, thr: torch.Tensor, stream=None) -> Tuple[SparseMap, torch.Tensor]:
    """spc_topk_keep_ge: the entries whose R7 composite >= thr[segment], in key order."""
    lib = load()
    ys = y.c_struct()
    ws = C.c_size_t()
    check("spc_topk_keep_query", lib.spc_topk_keep_query(C.byref(ys), C.byref(ws)))
    dev = y.values.device
    w = _workspace(ws.value, dev)
    keys, vals, nnz, o = _out(int(y.nnz_bound), dev)
    src = torch.empty(max(int(y.nnz_bound), 1), dtype=torch.int64, device=dev)
    check("spc_topk_keep_ge", lib.spc_topk_keep_ge(C.byref(ys), ATTN[attn], int(p_base), _ptr(thr), C.byref(o),
                                                   _ptr(src), _ptr(w), w.numel(), _stream(stream)))
    return SparseMap(keys, vals, y.batch, y.channels, y.dims, int(y.nnz_bound), nnz), src


# ------------------------------------------------------------------ communication
class Comm:
    """Collectives of the spatial layer over the ranks this process drives (`ranks`, in order).
    exchange(to_left, to_right): per local rank, lists of 1-D tensors sent to rank-1 / rank+1
    (None at the grid's ends); returns per local rank what rank-1 / rank+1 sent to it.
    allreduce_sum(ts): per local rank one tensor; afterwards each holds the sum over all ranks."""
    world: int
    ranks: List[int]

    def exchange(self, to_left, to_right):
        raise NotImplementedError

    def allreduce_sum(self, ts: List[torch.Tensor]):
        raise NotImplementedError


class LoopbackComm(Comm):
    """All `world` ranks in this process (virtual shards, lockstep)."""

    def __init__(self, world: int):
        self.world = int(world)
        self.ranks = list(range(self.world))

    def exchange(self, to_left, to_right):
        W = self.world
        from_left = [to_right[r - 1] if r > 0 else None for r in range(W)]
        from_right = [to_left[r + 1] if r < W - 1 else None for r in range(W)]
        return from_left, from_right

    def allreduce_sum(self, ts):
        tot = ts[0].clone()
        for t in ts[1:]:
            tot += t
        for t in ts:
            t.copy_(tot)


class DistComm(Comm):
    """One rank per process over torch.distributed (NCCL on GPUs, gloo in the CPU tests). With a
    gloo group and device tensors the payloads are staged through host memory (gloo has no
    device point-to-point): the multi-process tests on a single-GPU box use that."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]
        self.host_staging = dist.get_backend(group) == "gloo"

    def _p2p(self, sends, recv_shapes):
        """sends: [(peer, tensor)], recv_shapes: [(peer, n, dtype)] -> received tensors."""
        stage = self.host_staging
        outs, ops = [], []
        for peer, n, dt, dv in recv_shapes:
            t = torch.empty(n, dtype=dt, device="cpu" if stage else dv)
            outs.append(t)
            ops.append(dist.P2POp(dist.irecv, t, self._g(peer), self.group))
        for peer, t in sends:
            ops.append(dist.P2POp(dist.isend, t.contiguous().cpu() if stage else t.contiguous(), self._g(peer),
                                  self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if stage:
            outs = [t.to(dv) for t, (_, _, _, dv) in zip(outs, recv_shapes)]
        return outs

    def _g(self, peer: int) -> int:
        return peer if self.group is None else dist.get_global_rank(self.group, peer)

    def exchange(self, to_left, to_right):
        r, W = self.ranks[0], self.world
        tl, tr = to_left[0], to_right[0]
        ref = next(t for t in (tl or []) + (tr or []))
        dev = ref.device
        # 1. sizes (one int64 per tensor), 2. payloads
        nt = len(tl if tl is not None else tr)
        sends, shapes = [], []
        if r > 0:
            sends.append((r - 1, torch.tensor([t.numel() for t in tl], dtype=torch.int64, device=dev)))
            shapes.append((r - 1, nt, torch.int64, dev))
        if r < W - 1:
            sends.append((r + 1, torch.tensor([t.numel() for t in tr], dtype=torch.int64, device=dev)))
            shapes.append((r + 1, nt, torch.int64, dev))
        got = self._p2p(sends, shapes)
        sizes = {}
        i = 0
        if r > 0:
            sizes["l"] = got[i].tolist()
            i += 1
        if r < W - 1:
            sizes["r"] = got[i].tolist()
        sends, shapes = [], []
        dts = [t.dtype for t in (tl if tl is not None else tr)]
        if r > 0:
            sends += [(r - 1, t) for t in tl]
            shapes += [(r - 1, int(n), dt, dev) for n, dt in zip(sizes["l"], dts)]
        if r < W - 1:
            sends += [(r + 1, t) for t in tr]
            shapes += [(r + 1, int(n), dt, dev) for n, dt in zip(sizes["r"], dts)]
        got = self._p2p(sends, shapes)
        fl = got[:nt] if r > 0 else None
        fr = (got[nt:] if r > 0 else got[:nt]) if r < W - 1 else None
        return [fl], [fr]

    def allreduce_sum(self, ts):
        if self.host_staging and ts[0].is_cuda:
            h = ts[0].cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
            ts[0].copy_(h)
        else:
            dist.all_reduce(ts[0], op=dist.ReduceOp.SUM, group=self.group)


# ------------------------------------------------------------------ the layer
@dataclass
class _RankCtx:
    a: int
    e: int
    hl: int
    hr: int
    x_ext: SparseMap
    ext_idx: torch.Tensor
    n_from_left: int
    n_own: int
    n_from_right: int
    to_left_idx: Optional[torch.Tensor]
    to_right_idx: Optional[torch.Tensor]


class SpatialConv:
    """One sparse convolution layer (with optional attention) whose sample grids are split by
    planes across the ranks of `comm`. `planes` = the full grid's first dimension; the filter's
    ksize[0] // 2 halo planes must fit in every rank's range."""

    def __init__(self, comm: Comm, planes: int, timing: bool = False):
        self.comm = comm
        self.planes = int(planes)
        self.ctx: List[_RankCtx] = []
        # timing=True: CUDA events around every local rank's share of each phase (on the current
        # stream); rank_ms() = the GPU time each rank's own work took (with LoopbackComm the
        # ranks run one after the other, so this is what each GPU would spend computing)
        self.timing = bool(timing)
        self._ev: List[List[Tuple[torch.cuda.Event, torch.cuda.Event]]] = [[] for _ in comm.ranks]
        self.halo_bytes = [0 for _ in comm.ranks]

    def _t(self, j: int):
        layer = self

        class _Scope:
            def __enter__(self):
                if layer.timing:
                    self.a = torch.cuda.Event(enable_timing=True)
                    self.a.record()

            def __exit__(self, *exc):
                if layer.timing:
                    b = torch.cuda.Event(enable_timing=True)
                    b.record()
                    layer._ev[j].append((self.a, b))

        return _Scope()

    def rank_ms(self) -> List[float]:
        """Per local rank, the summed GPU time of its work since the last call (synchronises)."""
        torch.cuda.synchronize()
        out = [sum(a.elapsed_time(b) for a, b in ev) for ev in self._ev]
        self._ev = [[] for _ in self.comm.ranks]
        return out

    def ranges(self):
        return [plane_range(self.planes, self.comm.world, r) for r in self.comm.ranks]

    def forward(self, xs: List[SparseMap], w: SparseFilter, bias: Optional[torch.Tensor], attn: str = "magnitude",
                k: int = 0) -> List[SparseMap]:
        """xs: per local rank its shard of the input; returns per local rank its shard of the
        output (keys over the shard's planes; equal to the single-GPU layer's outputs there)."""
        h = int(w.ksize[0]) // 2
        W = self.comm.world
        rng = self.ranges()
        for (a, e) in rng:
            if e - a < max(h, 1):
                raise ValueError(f"spatial shard of {e - a} planes is thinner than the halo ({h})")
        # 1. boundary slabs for the neighbours
        to_left, to_right, tl_idx, tr_idx = [], [], [], []
        for j, (x, r, (a, e)) in enumerate(zip(xs, self.comm.ranks, rng)):
            with self._t(j):
                tl, il = self._slab(x, 0, h) if r > 0 and h > 0 else (None, None)
                tr, ir = self._slab(x, e - a - h, e - a) if r < W - 1 and h > 0 else (None, None)
            to_left.append(tl)
            tl_idx.append(il)
            to_right.append(tr)
            tr_idx.append(ir)
            self.halo_bytes[j] += sum(12 * int(t[0].numel()) for t in (tl, tr) if t is not None)
        if h > 0 and W > 1:
            from_left, from_right = self.comm.exchange(to_left, to_right)
        else:
            from_left = from_right = [None] * len(xs)
        # 2.-4. extended input, convolution, owned planes
        self.ctx = []
        ys = []
        for j, (x, (a, e)) in enumerate(zip(xs, rng)):
            n = e - a
            fl, fr = from_left[j], from_right[j]
            hl = h if fl is not None else 0
            hr = h if fr is not None else 0
            halo_dims = (h,) + tuple(x.dims[1:])
            with self._t(j):
                xe = x.exact()
                srcs = []
                if hl:
                    srcs.append((SparseMap(fl[0], fl[1], x.batch, x.channels, halo_dims, int(fl[0].numel())), 0, h, 0))
                srcs.append((xe, 0, n, hl))
                if hr:
                    srcs.append((SparseMap(fr[0], fr[1], x.batch, x.channels, halo_dims, int(fr[0].numel())), 0, h,
                                 hl + n))
                x_ext, ext_idx, _ = slab_gather(srcs, hl + n + hr, src_index=True)
                x_ext = x_ext.exact()
                y_ext = sparse_conv_fwd(x_ext, w, bias, "none", 0)
                y_own, _ = extract_planes(y_ext, hl, hl + n)
            self.ctx.append(_RankCtx(a, e, hl, hr, x_ext, ext_idx,
                                     int(fl[0].numel()) if hl else 0, xe.nnz_bound, int(fr[0].numel()) if hr else 0,
                                     tl_idx[j], tr_idx[j]))
            ys.append(y_own)
        if attn == "none":
            return ys
        return self._select(ys, attn, k)

    def _slab(self, x: SparseMap, lo: int, hi: int):
        m, i = extract_planes(x, lo, hi, src_index=True)
        m = m.exact()
        return [m.keys, m.values], i[:m.nnz_bound]

    def _select(self, ys: List[SparseMap], attn: str, k: int) -> List[SparseMap]:
        """5. exact k-selection per (b, oc) over all ranks' owned outputs."""
        if k < 1:
            raise ValueError("attention needs k >= 1")
        nseg = ys[0].batch * ys[0].channels
        plane = 1
        for d in ys[0].dims[1:]:
            plane *= int(d)
        if self.planes * plane > 2 ** 32:
            raise ValueError("the attention composite needs fewer than 2^32 positions per segment")
        sts = []
        for j, y in enumerate(ys):
            with self._t(j):
                sts.append(_select_init(nseg, k, y.values.device))
        for shift in range(56, -1, -8):
            for j, (y, st, c) in enumerate(zip(ys, sts, self.ctx)):
                with self._t(j):
                    _digit_hist(y, attn, c.a * plane, st, shift)
            self.comm.allreduce_sum([st.hist for st in sts])
            for j, st in enumerate(sts):
                with self._t(j):
                    _digit_pick(nseg, st, shift)
            # every rank holds the same summed histograms, hence the same settled flags: stop
            # once every segment's threshold is exact (usually after the score's bytes)
            if shift and not bool((sts[0].need >= 0).any()):
                break
        out = []
        for j, (y, st, c) in enumerate(zip(ys, sts, self.ctx)):
            with self._t(j):
                out.append(keep_ge(y, attn, c.a * plane, st.prefix)[0])
        return out

    def backward(self, xs: List[SparseMap], w: SparseFilter, ys: List[SparseMap], dys: List[torch.Tensor],
                 need_dx: bool = True):
        """Per local rank (dx of its input shard, dw, dbias); dw / dbias are the all-ranks sums
        (identical on every rank)."""
        nw = int(w.keys.numel())
        dev = xs[0].values.device
        parts, dxe = [], []
        # 6. local backward against the owned kept outputs
        for j, (y, dy, c) in enumerate(zip(ys, dys, self.ctx)):
            with self._t(j):
                ye = place_planes(y.exact(), c.hl, c.x_ext.dims[0]).exact()
                buf = torch.zeros(nw + w.c_out, dtype=torch.float64, device=dev)
                dx_ext = torch.empty(max(c.x_ext.nnz_bound, 1), dtype=torch.float32, device=dev) if need_dx else None
                BwdPlan(c.x_ext, w, ye).f64(c.x_ext, w, ye, dy, dx_ext, buf[:nw], buf[nw:])
            parts.append(buf)
            dxe.append(dx_ext)
        # 7. dw || dbias over ranks, one rounding
        self.comm.allreduce_sum(parts)
        dw = torch.empty(max(nw, 1), dtype=torch.float32, device=dev)
        db = torch.empty(w.c_out, dtype=torch.float32, device=dev)
        round_f64(parts[0][:nw], dw[:nw])
        round_f64(parts[0][nw:], db)
        if not need_dx:
            return [(None, dw[:nw], db) for _ in xs]
        # 7. the halo inputs' partials back to their owners
        dcats, to_left, to_right = [], [], []
        for j, (c, dx_ext) in enumerate(zip(self.ctx, dxe)):
            ntot = c.n_from_left + c.n_own + c.n_from_right
            with self._t(j):
                dcat = sparse_scatter_grad(c.ext_idx, dx_ext, c.x_ext.nnz_bound, ntot)
            dcats.append(dcat)
            to_left.append([dcat[:c.n_from_left]] if c.hl else None)
            to_right.append([dcat[c.n_from_left + c.n_own:ntot]] if c.hr else None)
        if self.comm.world > 1 and any(c.hl or c.hr for c in self.ctx):
            from_left, from_right = self.comm.exchange(to_left, to_right)
        else:
            from_left = from_right = [None] * len(xs)
        out = []
        for j, c in enumerate(self.ctx):
            with self._t(j):
                dx = dcats[j][c.n_from_left:c.n_from_left + c.n_own].clone()
                if from_left[j] is not None and c.to_left_idx is not None and c.to_left_idx.numel():
                    index_add(c.to_left_idx, from_left[j][0], dx)
                if from_right[j] is not None and c.to_right_idx is not None and c.to_right_idx.numel():
                    index_add(c.to_right_idx, from_right[j][0], dx)
            out.append((dx, dw[:nw], db))
        return out

"""Python binding of the C-ABI (same names as include/spconv.h). Marshalling only: every step
of the hot path runs in libspconv's CUDA kernels. PyTorch provides device memory and streams.

Sparse maps live on the device as (keys int64 [capacity], values float32 [capacity]) plus a
device nnz word; nothing here synchronises unless `.nnz()` / `.trimmed()` is called.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

import torch

from . import _lib
from ._lib import ATTN, VARIANT, DensityRegT, FilterT, MapOutT, MapT, check


def _stream(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


@dataclass
class SparseMap:
    """Device COO feature map: key = ((b*C + c)*V + row_major(p)) (include/spconv.h)."""

    keys: torch.Tensor          # int64 (bit pattern of the uint64 keys) or int32 ("Sparse 32"), [capacity]
    values: torch.Tensor        # float32 [capacity]
    batch: int
    channels: int
    dims: Tuple[int, ...]
    nnz_bound: int              # host upper bound (exact when nnz_dev is None)
    nnz_dev: Optional[torch.Tensor] = None   # int64 [1] exact count on the device

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def volume(self) -> int:
        v = 1
        for d in self.dims:
            v *= int(d)
        return v

    def nnz(self) -> int:
        """Exact count (synchronises when it lives on the device)."""
        return int(self.nnz_dev.item()) if self.nnz_dev is not None else int(self.nnz_bound)

    def trimmed(self) -> Tuple[torch.Tensor, torch.Tensor]:
        n = self.nnz()
        return self.keys[:n], self.values[:n]

    def exact(self) -> "SparseMap":
        """Same map with a host-exact nnz (synchronises once)."""
        n = self.nnz()
        return SparseMap(self.keys[:n], self.values[:n], self.batch, self.channels, self.dims, n, None)

    def c_struct(self) -> MapT:
        m = MapT()
        m.ndim = self.ndim
        m.batch = self.batch
        m.channels = self.channels
        for i, d in enumerate(self.dims):
            m.dims[i] = int(d)
        m.nnz = int(self.nnz_bound)
        m.nnz_dev = None if self.nnz_dev is None else self.nnz_dev.data_ptr()
        m.keys = self.keys.data_ptr() if self.keys.numel() else None
        m.values = self.values.data_ptr() if self.values.numel() else None
        m.key_bits = self.key_bits
        return m

    @property
    def key_bits(self) -> int:
        """32 for int32 key storage (Table 1 "Sparse 32"), else 64."""
        return 32 if self.keys.dtype == torch.int32 else 64

    def to_key_bits(self, bits: int) -> "SparseMap":
        """Same map with its keys stored in `bits` (32 / 64) bits (sparse_keys_narrow / _widen)."""
        if bits == self.key_bits:
            return self
        if bits == 32:
            k = keys_narrow(self)
        else:
            k = keys_widen(self.keys[:self.nnz_bound], self.nnz_bound, self.nnz_dev)
        return SparseMap(k, self.values, self.batch, self.channels, self.dims, self.nnz_bound, self.nnz_dev)

    @staticmethod
    def from_arrays(keys, values, batch: int, channels: int, dims: Sequence[int], device="cuda",
                    key_bits: int = 64) -> "SparseMap":
        """Upload host arrays (numpy uint64 keys / float32 values, or tensors); key_bits=32 stores
        the keys as int32 ("Sparse 32", valid below 2^32 keys)."""
        if not isinstance(keys, torch.Tensor):
            import numpy as np

            keys = np.ascontiguousarray(keys)
            keys = torch.from_numpy(keys.astype(np.uint32).view(np.int32) if key_bits == 32 else keys.view(np.int64))
        if not isinstance(values, torch.Tensor):
            values = torch.from_numpy(values)
        k = keys.to(device=device, dtype=torch.int32 if key_bits == 32 else torch.int64).contiguous()
        v = values.to(device=device, dtype=torch.float32).contiguous()
        return SparseMap(k, v, int(batch), int(channels), tuple(int(d) for d in dims), int(k.numel()), None)


@dataclass
class SparseFilter:
    """Device filter bank: key = ((oc*c_in + ic)*prod(ksize) + row_major(delta))."""

    keys: torch.Tensor
    values: torch.Tensor
    c_in: int
    c_out: int
    ksize: Tuple[int, ...]

    def c_struct(self) -> FilterT:
        f = FilterT()
        f.ndim = len(self.ksize)
        f.c_in = self.c_in
        f.c_out = self.c_out
        for i, k in enumerate(self.ksize):
            f.ksize[i] = int(k)
        f.nnz = int(self.keys.numel())
        f.keys = self.keys.data_ptr() if self.keys.numel() else None
        f.values = self.values.data_ptr() if self.values.numel() else None
        return f

    @staticmethod
    def from_arrays(keys, values, c_in: int, c_out: int, ksize: Sequence[int], device="cuda") -> "SparseFilter":
        if not isinstance(keys, torch.Tensor):
            import numpy as np

            keys = torch.from_numpy(np.ascontiguousarray(keys).view(np.int64))
        if not isinstance(values, torch.Tensor):
            values = torch.from_numpy(values)
        return SparseFilter(keys.to(device=device, dtype=torch.int64).contiguous(),
                            values.to(device=device, dtype=torch.float32).contiguous(),
                            int(c_in), int(c_out), tuple(int(k) for k in ksize))


def load():
    return _lib.load()


def version() -> str:
    return load().spc_version().decode()


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def _out(cap: int, device, key_bits: int = 64) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor, MapOutT]:
    keys = torch.empty(max(cap, 1), dtype=torch.int32 if key_bits == 32 else torch.int64, device=device)
    vals = torch.empty(max(cap, 1), dtype=torch.float32, device=device)
    nnz = torch.zeros(1, dtype=torch.int64, device=device)
    o = MapOutT()
    o.capacity = int(cap)
    o.keys = keys.data_ptr()
    o.values = vals.data_ptr()
    o.nnz_dev = nnz.data_ptr()
    o.key_bits = int(key_bits)
    return keys, vals, nnz, o


class FwdPlan:
    """Queries once, then reuses output and workspace buffers across calls with the same
    shapes (for timing loops and CUDA-graph capture).

    variant: "scatter" (S), "gemm" (G, tensor cores), "auto" (the library's cost model) or
    "measure" (time both once per layer shape and keep the faster: SURVEY §8 a3 "the faster
    variant is picked per layer from measurement")."""

    def __init__(self, x: SparseMap, w: SparseFilter, attn: str = "magnitude", k: int = 0, variant: str = "auto",
                 bias: Optional[torch.Tensor] = None, samples_per_pass: Optional[int] = None,
                 key_bits: Optional[int] = None):
        lib = load()
        self.attn = ATTN[attn]
        self.k = int(k)
        cap = C.c_int64()
        ws = C.c_size_t()
        xs, fs = x.c_struct(), w.c_struct()
        if samples_per_pass is None and variant in ("auto", "scatter", "measure"):
            samples_per_pass = _bounded_pass(lib, xs, fs, self.attn, self.k, x, variant)
        self.spp = samples_per_pass
        if samples_per_pass is not None:
            # batch-sliced scatter forward (spc_conv_fwd_query_pass): workspace for spp samples
            check("spc_conv_fwd_query_pass", lib.spc_conv_fwd_query_pass(C.byref(xs), C.byref(fs), self.attn, self.k,
                                                                         int(samples_per_pass), C.byref(cap),
                                                                         C.byref(ws)))
            self.variant = VARIANT["scatter"]
            self.resolved = "scatter"
        else:
            if variant == "measure":
                variant = select_variant(x, w, bias, attn, k)
            self.variant = VARIANT[variant]
            check("spc_conv_fwd_query_ex", lib.spc_conv_fwd_query_ex(C.byref(xs), C.byref(fs), self.attn, self.k,
                                                                     self.variant, C.byref(cap), C.byref(ws)))
            self.resolved = {1: "scatter", 2: "gemm"}.get(
                lib.spc_conv_fwd_variant(C.byref(xs), C.byref(fs), self.attn, self.k, self.variant), "?")
        dev = x.values.device
        self.capacity = int(cap.value)
        self.ws_bytes = int(ws.value)
        self.ws = _workspace(ws.value, dev)
        self.key_bits = x.key_bits if key_bits is None else int(key_bits)   # output keys: as the input by default
        self.keys, self.vals, self.nnz, self.out = _out(self.capacity, dev, self.key_bits)
        self.c_out = w.c_out
        self.batch, self.dims = x.batch, x.dims

    def __call__(self, x: SparseMap, w: SparseFilter, bias: Optional[torch.Tensor] = None,
                 stream: Optional[torch.cuda.Stream] = None) -> SparseMap:
        xs, fs = x.c_struct(), w.c_struct()
        if self.spp is not None:
            rc = load().sparse_conv_fwd_pass(C.byref(xs), C.byref(fs), _ptr(bias), self.attn, self.k, int(self.spp),
                                             C.byref(self.out), _ptr(self.ws), self.ws.numel(), _stream(stream))
            check("sparse_conv_fwd_pass", rc)
        else:
            rc = load().sparse_conv_fwd_ex(C.byref(xs), C.byref(fs), _ptr(bias), self.attn, self.k, self.variant,
                                           C.byref(self.out), _ptr(self.ws), self.ws.numel(), _stream(stream))
            check("sparse_conv_fwd_ex", rc)
        return SparseMap(self.keys, self.vals, self.batch, self.c_out, self.dims, self.capacity, self.nnz)


# Fraction of the free device memory the forward workspace may take before the batch is sliced
# into passes (sparse_conv_fwd_pass); SPC_FWD_MEM_FRAC overrides.
_WS_FRAC = float(os.environ.get("SPC_FWD_MEM_FRAC", "0.5"))


def _bounded_pass(lib, xs, fs, attn: int, k: int, x: "SparseMap", variant: str) -> Optional[int]:
    """None when the whole-batch forward's workspace fits _WS_FRAC of the free device memory;
    else the largest samples-per-pass whose workspace does (at least 1)."""
    cap, ws = C.c_int64(), C.c_size_t()
    v = VARIANT["scatter" if variant == "measure" else variant]
    if lib.spc_conv_fwd_query_ex(C.byref(xs), C.byref(fs), attn, k, v, C.byref(cap), C.byref(ws)) != 0:
        return None
    if not torch.cuda.is_available():
        return None
    free = torch.cuda.mem_get_info(x.values.device)[0]
    budget = _WS_FRAC * free
    if ws.value <= budget or x.batch <= 1:
        return None
    lo, hi = 1, int(x.batch) - 1   # largest spp with workspace <= budget
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if lib.spc_conv_fwd_query_pass(C.byref(xs), C.byref(fs), attn, k, mid, C.byref(cap), C.byref(ws)) == 0 \
                and ws.value <= budget:
            lo = mid
        else:
            hi = mid - 1
    return lo


_MEASURED = {}


def _layer_key(x: SparseMap, w: SparseFilter, attn: str, k: int):
    return (x.batch, x.channels, tuple(x.dims), w.c_out, tuple(w.ksize), int(w.keys.numel()),
            int(max(1, x.nnz_bound)).bit_length(), attn, int(k))


def select_variant(x: SparseMap, w: SparseFilter, bias=None, attn: str = "magnitude", k: int = 0, reps: int = 3) -> str:
    """Time the supported accumulate variants on this layer (CUDA events, after one warm-up call)
    and return the faster; cached per layer shape and input-size bucket."""
    key = _layer_key(x, w, attn, k)
    if key in _MEASURED:
        return _MEASURED[key]
    lib = load()
    xs, fs = x.c_struct(), w.c_struct()
    times = {}
    for name in ("scatter", "gemm"):
        cap, wsb = C.c_int64(), C.c_size_t()
        if lib.spc_conv_fwd_query_ex(C.byref(xs), C.byref(fs), ATTN[attn], int(k), VARIANT[name],
                                     C.byref(cap), C.byref(wsb)) != 0:
            continue
        plan = FwdPlan(x, w, attn, k, name)
        plan(x, w, bias)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            plan(x, w, bias)
        b.record()
        b.synchronize()
        times[name] = a.elapsed_time(b) / reps
        del plan
    choice = min(times, key=times.get) if times else "scatter"
    _MEASURED[key] = choice
    return choice


def sparse_conv_fwd(x: SparseMap, w: SparseFilter, bias: Optional[torch.Tensor] = None, attn: str = "magnitude",
                    k: int = 0, stream=None, variant: str = "auto", samples_per_pass: Optional[int] = None,
                    key_bits: Optional[int] = None) -> SparseMap:
    """Alg. 1. attn in {"none", "magnitude", "raw"}; k entries kept per (b, oc);
    variant in {"auto", "scatter", "gemm", "measure"} (FwdPlan); samples_per_pass bounds the
    workspace to that many samples' buffers (sparse_conv_fwd_pass, scatter variant); key_bits: the
    output's key width (default: the input's)."""
    return FwdPlan(x, w, attn, k, variant, bias, samples_per_pass, key_bits)(x, w, bias, stream)


class BwdPlan:
    def __init__(self, x: SparseMap, w: SparseFilter, y: SparseMap):
        lib = load()
        ws = C.c_size_t()
        xs, fs, ys = x.c_struct(), w.c_struct(), y.c_struct()
        check("spc_conv_bwd_query", lib.spc_conv_bwd_query(C.byref(xs), C.byref(fs), C.byref(ys), C.byref(ws)))
        self.ws = _workspace(ws.value, x.values.device)

    def __call__(self, x, w, y, dy, dx=None, dw=None, dbias=None, stream=None):
        xs, fs, ys = x.c_struct(), w.c_struct(), y.c_struct()
        lib = load()
        st = _stream(stream)
        if dbias is not None and dw is None:
            # dbias is produced with the weight gradient (sparse_conv_bwd / _weight); a scratch dw
            # keeps every requested output initialised
            dw = torch.empty(max(w.keys.numel(), 1), dtype=torch.float32, device=dbias.device)
        if dx is not None and dw is not None:
            rc = lib.sparse_conv_bwd(C.byref(xs), C.byref(fs), C.byref(ys), _ptr(dy), _ptr(dx), _ptr(dw), _ptr(dbias),
                                     _ptr(self.ws), self.ws.numel(), st)
            check("sparse_conv_bwd", rc)
        elif dx is not None:
            rc = lib.sparse_conv_bwd_input(C.byref(xs), C.byref(fs), C.byref(ys), _ptr(dy), _ptr(dx),
                                           _ptr(self.ws), self.ws.numel(), st)
            check("sparse_conv_bwd_input", rc)
        elif dw is not None:
            rc = lib.sparse_conv_bwd_weight(C.byref(xs), C.byref(fs), C.byref(ys), _ptr(dy), _ptr(dw), _ptr(dbias),
                                            _ptr(self.ws), self.ws.numel(), st)
            check("sparse_conv_bwd_weight", rc)
        return dx, dw, dbias


    def f64(self, x, w, y, dy, dx=None, dw64=None, dbias64=None, stream=None):
        """Data-parallel form (sparse_conv_bwd_f64): dx (fp32, optional) and the unrounded fp64
        accumulators of dw / dbias of this call (shard), to be summed across ranks and rounded
        once (dp.GradAllReduce)."""
        xs, fs, ys = x.c_struct(), w.c_struct(), y.c_struct()
        check("sparse_conv_bwd_f64", load().sparse_conv_bwd_f64(
            C.byref(xs), C.byref(fs), C.byref(ys), _ptr(dy), _ptr(dx), _ptr(dw64), _ptr(dbias64), _ptr(self.ws),
            self.ws.numel(), _stream(stream)))
        return dx, dw64, dbias64


def round_f64(src: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    """out = (float32) src, one rounding (spc_round_f64)."""
    n = int(src.numel())
    check("spc_round_f64", load().spc_round_f64(_ptr(src), _ptr(out), n, _stream(stream)))
    return out


def sparse_conv_bwd(x: SparseMap, w: SparseFilter, y: SparseMap, dy: torch.Tensor, need_dx=True, need_dw=True,
                    need_dbias=True, stream=None):
    """Alg. 2, Eqs. (3)/(4). Returns (dx [nnz_x], dw [nnz_w], dbias [c_out])."""
    dev = x.values.device
    dx = torch.empty(max(x.nnz_bound, 1), dtype=torch.float32, device=dev) if need_dx else None
    dw = torch.empty(max(w.keys.numel(), 1), dtype=torch.float32, device=dev) if need_dw else None
    db = torch.empty(w.c_out, dtype=torch.float32, device=dev) if need_dbias else None
    BwdPlan(x, w, y)(x, w, y, dy, dx, dw, db, stream)
    return (dx[:x.nnz_bound] if dx is not None else None, dw[:w.keys.numel()] if need_dw else None, db)


def sparse_conv_bwd_input(x, w, y, dy, stream=None):
    return sparse_conv_bwd(x, w, y, dy, True, False, False, stream)[0]


def sparse_conv_bwd_weight(x, w, y, dy, stream=None):
    _, dw, db = sparse_conv_bwd(x, w, y, dy, False, True, True, stream)
    return dw, db


def attention_topk(x: SparseMap, attn: str, k: int, stream=None) -> Tuple[SparseMap, torch.Tensor]:
    """Attention as a standalone layer. Returns (kept map, src index)."""
    lib = load()
    cap = C.c_int64()
    ws = C.c_size_t()
    xs = x.c_struct()
    a = ATTN[attn]
    check("spc_topk_query", lib.spc_topk_query(C.byref(xs), a, int(k), C.byref(cap), C.byref(ws)))
    dev = x.values.device
    keys, vals, nnz, o = _out(int(cap.value), dev, x.key_bits)
    src = torch.empty(max(int(cap.value), 1), dtype=torch.int64, device=dev)
    w = _workspace(ws.value, dev)
    check("attention_topk", lib.attention_topk(C.byref(xs), a, int(k), C.byref(o), _ptr(src), _ptr(w), w.numel(),
                                               _stream(stream)))
    return SparseMap(keys, vals, x.batch, x.channels, x.dims, int(cap.value), nnz), src


def sparse_relu(x: SparseMap, stream=None) -> Tuple[SparseMap, torch.Tensor]:
    """Sparse ReLU. Returns (kept map, src index)."""
    lib = load()
    cap = C.c_int64()
    ws = C.c_size_t()
    xs = x.c_struct()
    check("spc_relu_query", lib.spc_relu_query(C.byref(xs), C.byref(cap), C.byref(ws)))
    dev = x.values.device
    keys, vals, nnz, o = _out(int(cap.value), dev, x.key_bits)
    src = torch.empty(max(int(cap.value), 1), dtype=torch.int64, device=dev)
    w = _workspace(ws.value, dev)
    check("sparse_relu", lib.sparse_relu(C.byref(xs), C.byref(o), _ptr(src), _ptr(w), w.numel(), _stream(stream)))
    return SparseMap(keys, vals, x.batch, x.channels, x.dims, int(cap.value), nnz), src


def sparse_maxpool(x: SparseMap, stride: Sequence[int], stream=None) -> Tuple[SparseMap, torch.Tensor]:
    """Sparse max-pooling (§3.3). Returns (pooled map with dims ceil(d/s), argmax index)."""
    lib = load()
    cap = C.c_int64()
    ws = C.c_size_t()
    xs = x.c_struct()
    st = (C.c_int64 * len(stride))(*[int(s) for s in stride])
    check("spc_maxpool_query", lib.spc_maxpool_query(C.byref(xs), C.cast(st, C.c_void_p), C.byref(cap), C.byref(ws)))
    dev = x.values.device
    keys, vals, nnz, o = _out(int(cap.value), dev, x.key_bits)
    arg = torch.empty(max(int(cap.value), 1), dtype=torch.int64, device=dev)
    w = _workspace(ws.value, dev)
    check("sparse_maxpool", lib.sparse_maxpool(C.byref(xs), C.cast(st, C.c_void_p), C.byref(o), _ptr(arg), _ptr(w),
                                               w.numel(), _stream(stream)))
    pdims = tuple(-(-int(d) // int(s)) for d, s in zip(x.dims, stride))
    return SparseMap(keys, vals, x.batch, x.channels, pdims, int(cap.value), nnz), arg


def sparse_scatter_grad(src: torch.Tensor, dy: torch.Tensor, n_out_bound: int, n_in: int,
                        n_out_dev: Optional[torch.Tensor] = None, stream=None, sorted: bool = False) -> torch.Tensor:
    """Backward of ReLU / pool / top-k (Eq. (5)): dx[src[t]] = dy[t], zeros elsewhere.
    sorted=True (src strictly increasing: ReLU, top-k) takes sparse_scatter_grad_sorted."""
    dx = torch.empty(max(n_in, 1), dtype=torch.float32, device=dy.device)
    fn = "sparse_scatter_grad_sorted" if sorted else "sparse_scatter_grad"
    check(fn, getattr(load(), fn)(_ptr(src), _ptr(dy), int(n_out_bound), _ptr(n_out_dev), _ptr(dx), int(n_in),
                                  _stream(stream)))
    return dx[:n_in]


# ------------------------------------------------------------------ instrumentation
def kernel_launches() -> int:
    """Kernels launched by libspconv so far in this process."""
    return int(load().spc_kernel_launches())


def profile_enable(on: bool = True):
    load().spc_profile_enable(1 if on else 0)


def profile_reset():
    load().spc_profile_reset()


def profile_read():
    """{phase: (total_ms, launches)} of the CUDA-event brackets recorded while enabled."""
    import numpy as np

    n = 64
    names = C.create_string_buffer(8192)
    ms = np.zeros(n, np.float64)
    cnt = np.zeros(n, np.int64)
    k = load().spc_profile_read(names, 8192, ms.ctypes.data_as(C.c_void_p), cnt.ctypes.data_as(C.c_void_p), n)
    labels = names.raw.split(b"\0")[:k]
    return {lab.decode(): (float(ms[i]), int(cnt[i])) for i, lab in enumerate(labels)}


# ------------------------------------------------------------------ training-loop steps (f1)
@dataclass
class DensityReg:
    """Eq. (6) parameters of the adaptive density regulariser (§3.5); the paper uses 0.1 each."""

    lam: float
    rho_up: float
    o: float = 0.1
    b1: float = 0.1
    b2: float = 0.1


def adagrad_step(params: torch.Tensor, grad: torch.Tensor, accum: torch.Tensor, lr: float, eps: float = 1e-8,
                 reg: Optional[DensityReg] = None, y: Optional[SparseMap] = None, stream=None) -> None:
    """In-place Adagrad step over stored parameters (§4) with the density regulariser (§3.5); the
    layer density is y's device count over its cells (no host sync). sparse_adagrad_step."""
    n = int(params.numel())
    r = None
    ynnz, cells = None, 0.0
    if reg is not None:
        if y is None or y.nnz_dev is None:
            raise ValueError("the density regulariser needs the layer output y with a device count")
        r = DensityRegT(reg.lam, reg.rho_up, reg.o, reg.b1, reg.b2)
        ynnz, cells = C.c_void_p(y.nnz_dev.data_ptr()), float(y.batch * y.channels * y.volume)
    rc = load().sparse_adagrad_step(_ptr(params), _ptr(grad), _ptr(accum), n, ynnz, cells,
                                    C.byref(r) if r is not None else None, float(lr), float(eps), _stream(stream))
    check("sparse_adagrad_step", rc)


def filter_prune(w: SparseFilter, accum: Optional[torch.Tensor], warn: torch.Tensor, eps: float = 0.01,
                 stream=None) -> Tuple[SparseFilter, Optional[torch.Tensor], torch.Tensor]:
    """One-warning-shot pruning at an epoch end (§3.6): returns the compacted filter, its
    Adagrad accumulators and warning flags (synchronises once to learn the new count)."""
    lib = load()
    n = int(w.keys.numel())
    wsb = C.c_size_t()
    check("spc_prune_query", lib.spc_prune_query(n, C.byref(wsb)))
    dev = w.values.device
    ws = _workspace(wsb.value, dev)
    ok = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    ov = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    oa = torch.empty(max(n, 1), dtype=torch.float32, device=dev) if accum is not None else None
    ow = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    nnz = torch.zeros(1, dtype=torch.int64, device=dev)
    rc = lib.sparse_filter_prune(_ptr(w.keys), _ptr(w.values), _ptr(accum), _ptr(warn), n, float(eps), _ptr(ok),
                                 _ptr(ov), _ptr(oa), _ptr(ow), _ptr(nnz), _ptr(ws), ws.numel(), _stream(stream))
    check("sparse_filter_prune", rc)
    m = int(nnz.item())
    wf = SparseFilter(ok[:m].clone(), ov[:m].clone(), w.c_in, w.c_out, w.ksize)
    return wf, (oa[:m].clone() if oa is not None else None), ow[:m].clone()


# ------------------------------------------------------------------ sparseToDense bridge (f3)
def sparse_to_dense(x: SparseMap, stream=None) -> torch.Tensor:
    """Table 2 sparseToDense(): dense [batch, channels, *dims] tensor, zeros off the map."""
    dense = torch.empty((x.batch, x.channels) + tuple(x.dims), dtype=torch.float32, device=x.values.device)
    xs = x.c_struct()
    check("sparse_to_dense", load().sparse_to_dense(C.byref(xs), _ptr(dense), _stream(stream)))
    return dense


def sparse_to_dense_bwd(x: SparseMap, ddense: torch.Tensor, stream=None) -> torch.Tensor:
    """Gradient of sparse_to_dense w.r.t. the stored values: ddense at the stored keys."""
    dv = torch.empty(max(x.nnz_bound, 1), dtype=torch.float32, device=ddense.device)
    xs = x.c_struct()
    check("sparse_to_dense_bwd", load().sparse_to_dense_bwd(C.byref(xs), _ptr(ddense.contiguous()), _ptr(dv),
                                                            _stream(stream)))
    return dv[:x.nnz_bound]


# ------------------------------------------------------------------ key codec
def _dims_arg(dims):
    arr = (C.c_int64 * len(dims))(*[int(d) for d in dims])
    return C.cast(arr, C.c_void_p), arr   # (pointer, owner kept alive by the caller)


def encode_keys(coords: torch.Tensor, batch: int, channels: int, dims, stream=None) -> torch.Tensor:
    """spc_encode_keys: int64 coordinate rows (b, c, p_0..) [n, 2 + ndim] on the device -> uint64
    keys (as int64) [n]; raises ValueError when a coordinate is out of range."""
    coords = coords.contiguous()
    n = coords.shape[0]
    keys = torch.empty(max(n, 1), dtype=torch.int64, device=coords.device)
    bad = torch.zeros(1, dtype=torch.int32, device=coords.device)
    dp, _own = _dims_arg(dims)
    check("spc_encode_keys", load().spc_encode_keys(len(dims), int(batch), int(channels), dp,
                                                    _ptr(coords), n, _ptr(keys), _ptr(bad), _stream(stream)))
    if int(bad.item()):
        raise ValueError("spc_encode_keys: coordinate out of range")
    return keys[:n]


def decode_keys(keys: torch.Tensor, batch: int, channels: int, dims, stream=None) -> torch.Tensor:
    """spc_decode_keys: uint64 keys (as int64) [n] -> int64 coordinate rows (b, c, p_0..) [n, 2 + ndim];
    raises ValueError when a key is outside the key space."""
    keys = keys.contiguous()
    n = keys.shape[0]
    coords = torch.empty((max(n, 1), 2 + len(dims)), dtype=torch.int64, device=keys.device)
    bad = torch.zeros(1, dtype=torch.int32, device=keys.device)
    dp, _own = _dims_arg(dims)
    check("spc_decode_keys", load().spc_decode_keys(len(dims), int(batch), int(channels), dp,
                                                    _ptr(keys), n, _ptr(coords), _ptr(bad), _stream(stream)))
    if int(bad.item()):
        raise ValueError("spc_decode_keys: key outside the key space")
    return coords[:n]


# ------------------------------------------------------------------ memory model
def memory_estimate(ndim: int, r: int, batch: int, channels: int, rho_up: float, index_bits: int = 64) -> dict:
    """Table 1 / Fig. 7 theoretical bytes (spc_memory_estimate): dense, sparse, temp."""
    d, sp, t = C.c_double(), C.c_double(), C.c_double()
    check("spc_memory_estimate", load().spc_memory_estimate(int(ndim), int(r), int(batch), int(channels),
                                                            float(rho_up), int(index_bits), C.byref(d),
                                                            C.byref(sp), C.byref(t)))
    return {"dense": d.value, "sparse": sp.value, "temp": t.value}


def keys_narrow(x: SparseMap, stream=None) -> torch.Tensor:
    """Table 1 "Sparse 32" storage: int32 tensor holding the low 32 bits of every key."""
    out = torch.empty(max(x.nnz_bound, 1), dtype=torch.int32, device=x.keys.device)
    xs = x.c_struct()
    check("sparse_keys_narrow", load().sparse_keys_narrow(C.byref(xs), _ptr(out), _stream(stream)))
    return out[:x.nnz_bound]


def keys_widen(keys32: torch.Tensor, nnz_bound: int, nnz_dev: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """Inverse of keys_narrow: int64 keys (zero-extended)."""
    out = torch.empty(max(nnz_bound, 1), dtype=torch.int64, device=keys32.device)
    check("sparse_keys_widen", load().sparse_keys_widen(_ptr(keys32), _ptr(nnz_dev), int(nnz_bound), _ptr(out),
                                                        _stream(stream)))
    return out[:nnz_bound]

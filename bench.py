#!/usr/bin/env python
"""bench.py — sparse conv fwd+bwd on B200 (BASELINE.json metric, configs[3] = C4).

Workload (N=1): 3D 128^3 grid, batch 64, 8 -> 8 channels, 3x3x3 filters pruned to 50%
(rho_f = 0.5), input density rho_d per (b, c) (default 2%; --density), attention with
rho_up = 5% (k = floor(0.05 * 128^3) = 104857 per (b, oc), magnitude variant). One step =
sparse_conv_fwd (Alg. 1 with attention) + sparse_conv_bwd (Alg. 2: dx, dw, dbias) [+ NCCL
all-reduce of dw||dbias when N > 1]. With N GPUs the global batch of 64 is sharded (strong
scaling, BASELINE "batch 64 sharded on 1/2/4/8 GPUs").

Metric: effective GMAC/s = algorithmic MACs / time, where fwd MACs are the in-bounds
(input, weight) pairs (Eq. (1) first term) and bwd MACs are 2 x the pairs landing on
kept outputs (dx and dw). HBM GB/s is reported alongside from compulsory bytes.

  python bench.py [--gpus N --steps K --warmup W] [--density 0.02] [--impl reference]
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import uniform_map, sparse_filter, bias_vector, grad_values, select_samples, SEED_BASE  # noqa: E402

RES = 128
BATCH = 64
C_IN = C_OUT = 8
KS = (3, 3, 3)
RHO_F = 0.5
RHO_UP = 0.05
K_SEL = int(RHO_UP * RES ** 3)           # 104857 (reading R5: floor)
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def c4_inputs(density: float = 0.02, values: str = "continuous", batch: int = BATCH, b0: int = 0):
    """Seeded C4 inputs (per-sample streams: a shard generates only its own samples)."""
    seed = SEED_BASE * 1000 + 400 + int(round(density * 1000))
    x = uniform_map(batch, C_IN, (RES,) * 3, density, seed, values=values, b0=b0)
    w = sparse_filter(C_IN, C_OUT, KS, RHO_F, SEED_BASE + 4, values=values)
    bias = bias_vector(C_OUT, SEED_BASE + 4, values=values)
    return dict(x=x, w=w, bias=bias, k=K_SEL, density=density)


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region (NVML every 2 ms; the
    nvidia-smi fields of the profiling recipe's clocks line)."""
    REASONS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop = threading.Event()
        self.thread = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            idx = int(vis.split(",")[self.index]) if vis and vis.split(",")[0].isdigit() else self.index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv = pynvml
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def _sample(self):
        nv = self.nv
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
        self.mx.append(float(self.max_sm))
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        for name, bit in self.REASONS.items():
            if bits & bit:
                self.reasons.add(name)

    def _run(self):
        while not self.stop.wait(0.002):
            try:
                self._sample()
            except Exception:
                return

    def __exit__(self, *a):
        if self.thread:
            self.stop.set()
            self.thread.join(timeout=2)
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx),
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


# ----------------------------------------------------------------- MAC accounting
def algorithmic_macs(torch, X, W, y_keys_list, B_local, V):
    """Exact Eq. (1) MAC count: per output (b, oc, p) the number of in-bounds (input, weight)
    pairs = dense correlation of the occupancy masks (integer-valued, exact in fp32). fwd = sum
    over all p; bwd = 2 x sum over the kept p (dx and dw). Measurement plumbing only."""
    import torch.nn.functional as F

    dev = X.values.device
    wmask = torch.zeros(C_OUT * C_IN * 27, device=dev)
    wmask[W.keys.long()] = 1.0
    wmask = wmask.view(C_OUT, C_IN, 3, 3, 3)
    fwd = 0
    kept = 0
    keys = X.keys[:X.nnz_bound]
    ykeys = y_keys_list
    old = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False
    step = 4
    for b0 in range(0, B_local, step):
        nb = min(step, B_local - b0)
        lo = b0 * C_IN * V
        hi = (b0 + nb) * C_IN * V
        sel = keys[(keys >= lo) & (keys < hi)] - lo
        m = torch.zeros(nb * C_IN * V, device=dev)
        m[sel] = 1.0
        cnt = F.conv3d(m.view(nb, C_IN, RES, RES, RES), wmask, padding=1)
        fwd += int(cnt.double().sum().item())
        ylo, yhi = b0 * C_OUT * V, (b0 + nb) * C_OUT * V
        ys = ykeys[(ykeys >= ylo) & (ykeys < yhi)] - ylo
        kept += int(cnt.reshape(-1)[ys].double().sum().item())
        del m, cnt
    torch.backends.cudnn.allow_tf32 = old
    return fwd, 2 * kept


# ----------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1801_10585_b200 as spc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spc.load()
    assert BATCH % world == 0
    B_local = BATCH // world
    b0 = rank * B_local
    V = RES ** 3
    cfg = c4_inputs(args.density, args.values, batch=B_local, b0=b0)
    x, w, bias, k = cfg["x"], cfg["w"], cfg["bias"], cfg["k"]
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
    W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
    bias_t = torch.from_numpy(bias).cuda()
    fwd = spc.FwdPlan(X, W, "magnitude", k, args.variant, bias_t, args.samples_per_pass)
    args.resolved_variant = fwd.resolved
    cap = fwd.capacity
    dy_t = torch.from_numpy(grad_values(cap, SEED_BASE + 7 + rank)).cuda()
    Y0 = fwd(X, W, bias_t)
    bwd = spc.BwdPlan(X, W, Y0)
    dx_t = torch.empty(max(X.nnz_bound, 1), device="cuda")
    dw_t = torch.empty(W.keys.numel(), device="cuda")
    db_t = torch.empty(C_OUT, device="cuda")
    allreduce = spc.dp.GradAllReduce(W.keys.numel(), C_OUT, "cuda")   # SUM of dw||dbias (R13)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # 512 MB > L2

    def step():
        Y = fwd(X, W, bias_t)
        bwd(X, W, Y, dy_t, dx_t, dw_t, db_t)
        allreduce(dw_t, db_t)               # no-op on one GPU
        return Y

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # algorithmic work of one step (measurement plumbing, outside the timed region)
    Y = step()
    torch.cuda.synchronize()
    ny = int(Y.nnz_dev.item())
    fwd_macs, bwd_macs = algorithmic_macs(torch, X, W, Y.keys[:ny], B_local, V)
    nnz_x, nnz_w = x.nnz, w.nnz
    fwd_bytes = 12 * nnz_x + 12 * nnz_w + 4 * C_OUT + 12 * ny
    bwd_bytes = 12 * nnz_x + 4 * nnz_x + 12 * ny + 16 * nnz_w
    launches0 = spc.kernel_launches()
    step()
    torch.cuda.synchronize()
    launches_per_step = spc.kernel_launches() - launches0

    # ---- timed region: K steps, L2 flushed between steps (not timed), CUDA events
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record()
            step()
            evs[i][1].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    per_step = [a.elapsed_time(b) for a, b in evs]
    t_ms = float(sum(per_step))
    if world > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
        tot = torch.tensor([fwd_macs + bwd_macs, fwd_bytes + bwd_bytes], dtype=torch.float64, device="cuda")
        dist.all_reduce(tot)
        macs_all, bytes_all = float(tot[0].item()), float(tot[1].item())
    else:
        macs_all, bytes_all = float(fwd_macs + bwd_macs), float(fwd_bytes + bwd_bytes)
    ms_per_step = t_ms / args.steps
    value = macs_all / (ms_per_step * 1e-3) / 1e9

    # ---- per-kernel durations (CUDA events the library records on its stream)
    spc.profile_reset()
    spc.profile_enable(True)
    nprof = max(1, min(3, args.steps))
    for _ in range(nprof):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    prof = spc.profile_read()
    spc.profile_enable(False)
    phases = {k2: {"ms_per_step": v[0] / nprof, "launches_per_step": v[1] / nprof} for k2, v in prof.items()}
    step_sum = sum(p["ms_per_step"] for p in phases.values()) or 1.0
    top = max(phases, key=lambda n: phases[n]["ms_per_step"])
    pk, src = peaks()
    roof = roofline_for(top, phases[top], ny, nnz_x, nnz_w, B_local, fwd_macs, bwd_macs, pk, src, clk.summary())
    roof["share_of_step"] = phases[top]["ms_per_step"] / step_sum

    # ---- end to end through the C-ABI with host buffers (pinned), copies inside the region
    e2e = run_e2e(torch, spc, x, w, bias, k, cap, dy_t, args, world, dist if world > 1 else None)

    result = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline(cfg, fwd_macs, bwd_macs, Y, x)
        e2e_value = (macs_all / (e2e["ms_per_step"] * 1e-3) / 1e9) if e2e else None
        result = {
            "metric": "sparse conv fwd+bwd effective GMAC/s (C4 128^3, rho_up 5%)",
            "value": round(value, 3),
            "unit": "GMAC/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": f"synthetic ({args.values} values, uniform positions, seeded)",
            "config": {
                "workload": f"C4: 3D {RES}^3, batch {BATCH} (sharded {B_local}/GPU), {C_IN}->{C_OUT} ch, 3x3x3, "
                            f"rho_f {RHO_F}, rho_d {args.density}, rho_up {RHO_UP} (k={K_SEL}), magnitude attention, "
                            f"fwd + bwd(dx,dw,dbias)",
                "global_batch": BATCH,
                "density": args.density,
                "fwd_variant": f"{args.variant} -> {args.resolved_variant}",
                "fwd_samples_per_pass": args.samples_per_pass or "all",
                "fwd_workspace_gb": round(fwd.ws_bytes / 1e9, 3),
                "parallelism": f"dp{world}",
                "l2": "flushed between timed steps (512 MB write); inputs also exceed L2",
            },
            "hbm_gbs": round(bytes_all / (ms_per_step * 1e-3) / 1e9, 2),
            "work_per_step": {"fwd_macs": fwd_macs, "bwd_macs": bwd_macs, "nnz_x": nnz_x, "nnz_w": nnz_w,
                              "nnz_y": ny, "compulsory_bytes": fwd_bytes + bwd_bytes},
            "per_step_ms": [round(t, 4) for t in per_step],
            "kernels": {n: {"ms": round(p["ms_per_step"], 4), "n": p["launches_per_step"],
                            "share": round(p["ms_per_step"] / step_sum, 4)} for n, p in
                        sorted(phases.items(), key=lambda kv: -kv[1]["ms_per_step"])},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 3) if e2e_value else None, "unit": "GMAC/s",
                    "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                    "ms_per_step": round(e2e["ms_per_step"], 4)} if e2e else None,
            "gpu_launches": int(launches_per_step * args.steps),
            "gpu_launches_per_step": int(launches_per_step),
            "clocks": clk.summary(),
        }
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


def roofline_for(name, ph, ny, nnz_x, nnz_w, B_local, fwd_macs, bwd_macs, pk, src, clocks):
    """Roofline of the dominant kernel: algorithmic work per launch over the
    average launch duration = the step's work over the kernel's time per step (the batch-sliced
    forward launches the kernel once per pass, each on 1/passes of the work)."""
    t = ph["ms_per_step"] * 1e-3
    V = RES ** 3
    nseg = B_local * C_OUT
    hbm = float(pk.get("hbm_gbs", 6650.0))
    sm_mhz = float(pk.get("sm_max_mhz", 1965.0))
    # The scatter convolutions are bound by shared-memory read-modify-writes, not by FFMA issue:
    # every MAC of Alg. 1 (fwd) reads and writes one 4-byte accumulator word (8 B through the
    # 128 B/clk/SM shared-memory crossbar, B300_MICROARCH "LDS/STS"), so the peak is 16 MAC/clk/SM.
    # The backward reads one 4-byte gradient word per (entry, weight) pair it visits (every pair
    # is visited; 2 MACs are algorithmic only on kept outputs): 32 pair visits/clk/SM on the same
    # crossbar. DESIGN.md section 7 derives both.
    lsu_fwd = 148 * 16 * sm_mhz * 1e6 / 1e12
    if name == "conv_fwd":
        return {"kernel": name, "bound": "alu", "achieved": round(fwd_macs / t / 1e12, 4), "unit": "TMAC/s",
                "peak": round(lsu_fwd, 3), "frac": round(fwd_macs / t / 1e12 / lsu_fwd, 4),
                "traffic": ncu_traffic(name),
                "peak_source": f"derived: shared-memory RMW rate 148 SM x 128 B/clk / 8 B per MAC x {sm_mhz:.0f} MHz",
                "algorithmic": f"{fwd_macs} MACs per step (Eq. (1) pairs) in {ph['launches_per_step']:g} launch(es)"}
    if name == "conv_bwd":
        lsu_bwd = 148 * 32 * sm_mhz * 1e6 / 1e12   # pair visits/s: one 4-byte G load each
        return {"kernel": name, "bound": "alu", "achieved": round(fwd_macs / t / 1e12, 4), "unit": "Tpair/s",
                "peak": round(lsu_bwd, 3), "frac": round(fwd_macs / t / 1e12 / lsu_bwd, 4),
                "traffic": ncu_traffic(name),
                "peak_source": f"derived: one 4-byte shared gradient load per (entry, weight) pair, 148 SM x 32 lanes/clk x {sm_mhz:.0f} MHz",
                "algorithmic": f"{fwd_macs} (entry, weight) pairs visited per step ({bwd_macs} MACs on kept outputs) in {ph['launches_per_step']:g} launch(es)"}
    per_launch_bytes = {
        "fwd_classify": 4 * nseg * V,
        "fwd_write": 4 * nseg * V + 12 * ny,
        "row_index": 8 * nnz_x + 4 * (B_local * C_IN * RES * RES + 1),
        "dbias": 12 * ny,
    }.get(name)
    if per_launch_bytes is None:
        return {"kernel": name, "bound": "unknown", "achieved": None, "peak": None, "unit": None, "frac": None,
                "traffic": None}
    gbs = per_launch_bytes / t / 1e9
    return {"kernel": name, "bound": "hbm", "achieved": round(gbs, 1), "unit": "GB/s", "peak": hbm,
            "frac": round(gbs / hbm, 4), "traffic": ncu_traffic(name),
            "peak_source": f"{src} (MEASURED_PEAKS.json hbm_gbs)",
            "algorithmic": f"{per_launch_bytes} bytes per step in {ph['launches_per_step']:g} launch(es)"}


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full capture, or None."""
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_traffic.json")), reverse=True):
        try:
            d = json.load(open(path))
        except Exception:
            continue
        if kernel in d:
            return {"bytes": d[kernel]["traffic"], "source": os.path.relpath(path, ROOT) + ":" + d[kernel]["report"]}
    return None


def run_e2e(torch, spc, x, w, bias, k, cap, dy_dev, args, world, dist):
    """Same step through the public API with HOST inputs: every step's inputs (x keys/values, dy)
    are copied H2D from pinned memory inside the timed region and its result (dw, dbias, output
    nnz) is read back D2H. Like a data loader, the upload of step i+1 runs on a copy stream into
    the second of two device input buffers while step i computes (the buffer is reused only after
    the step that read it has finished)."""
    hk = torch.from_numpy(x.keys.view(np.int64)).pin_memory()
    hv = torch.from_numpy(x.values).pin_memory()
    hdy = dy_dev.cpu().pin_memory()
    bufs = [(torch.empty_like(hk, device="cuda"), torch.empty_like(hv, device="cuda"),
             torch.empty_like(hdy, device="cuda")) for _ in range(2)]
    W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
    bias_t = torch.from_numpy(bias).cuda()
    Xs = [spc.SparseMap(bk, bv, x.batch, x.channels, x.dims, x.nnz, None) for bk, bv, _ in bufs]
    fwd = spc.FwdPlan(Xs[0], W, "magnitude", k, args.resolved_variant, None, args.samples_per_pass)
    for bk, bv, bd in bufs:
        bk.copy_(hk)
        bv.copy_(hv)
        bd.copy_(hdy)
    Y0 = fwd(Xs[0], W, bias_t)
    bwd = spc.BwdPlan(Xs[0], W, Y0)
    dx = torch.empty(max(x.nnz, 1), device="cuda")
    dw = torch.empty(W.keys.numel(), device="cuda")
    db = torch.empty(C_OUT, device="cuda")
    out_dw = torch.empty(W.keys.numel()).pin_memory()
    out_db = torch.empty(C_OUT).pin_memory()
    out_n = torch.empty(1, dtype=torch.int64).pin_memory()
    allreduce = spc.dp.GradAllReduce(W.keys.numel(), C_OUT, "cuda")
    comp = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    loaded = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]

    def upload(i):
        j = i % 2
        with torch.cuda.stream(copy):
            copy.wait_event(consumed[j])         # the step that last read buffer j is done
            bk, bv, bd = bufs[j]
            bk.copy_(hk, non_blocking=True)
            bv.copy_(hv, non_blocking=True)
            bd.copy_(hdy, non_blocking=True)
            loaded[j].record(copy)

    def step(i, last):
        j = i % 2
        if not last:
            upload(i + 1)
        comp.wait_event(loaded[j])
        Y = fwd(Xs[j], W, bias_t)
        bwd(Xs[j], W, Y, bufs[j][2], dx, dw, db)
        consumed[j].record(comp)
        allreduce(dw, db)
        out_dw.copy_(dw, non_blocking=True)
        out_db.copy_(db, non_blocking=True)
        out_n.copy_(Y.nnz_dev, non_blocking=True)

    def run(n):
        for e in consumed:
            e.record(comp)
        upload(0)
        for i in range(n):
            step(i, i == n - 1)

    run(max(1, args.warmup))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = max(1, args.steps)
    if dist is not None:
        dist.barrier()
    e0.record()
    run(n)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    if dist is not None:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    return {"ms_per_step": ms, "h2d": int(hk.numel() * 8 + hv.numel() * 4 + hdy.numel() * 4),
            "d2h": int(out_dw.numel() * 4 + out_db.numel() * 4 + 8)}


# --------------------------------------------------------------------- CPU baseline
def cpu_baseline(cfg, fwd_macs_total, bwd_macs_total, Y, x):
    """The oracle (oracle/, plain C, fp64, single thread) on one sample of the same workload."""
    import oracle as ora

    xs = select_samples(x, [0])
    t0 = time.perf_counter()
    yk, yv, _, macs = ora.conv_fwd(xs, cfg["w"], cfg["bias"], attn=ora.ATTN_MAGNITUDE, k=cfg["k"])
    dy = grad_values(yk.shape[0], SEED_BASE + 99)
    *_, kept_pairs = ora.conv_bwd(xs, cfg["w"], yk, dy, return_pairs=True)
    dt = time.perf_counter() - t0
    bwd = 2 * kept_pairs
    return {"value": round((macs + bwd) / dt / 1e9, 4), "unit": "GMAC/s", "cores": 1, "kind": "oracle",
            "sample": f"1 of {BATCH} samples (b=0), fwd+bwd, {dt:.1f} s", "seconds": round(dt, 2)}


# ------------------------------------------------------------------- reference arm
def run_reference(args):
    """--impl reference: the oracle as it stands, on this host's cores, on the same config and
    metric. Each step = fwd+bwd of one (b, oc) pair of the C4 workload (a bounded sample)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import oracle as ora
    from synth import Filter

    cfg = c4_inputs(args.density, args.values, batch=1)
    x, w = cfg["x"], cfg["w"]
    V = RES ** 3

    def one(oc):
        KV = 27
        lo, hi = np.searchsorted(w.keys, np.uint64(oc * C_IN * KV)), np.searchsorted(w.keys, np.uint64((oc + 1) * C_IN * KV))
        wk = w.keys[lo:hi] - np.uint64(oc * C_IN * KV)
        wo = Filter(C_IN, 1, KS, wk, w.values[lo:hi])
        t0 = time.perf_counter()
        yk, yv, _, macs = ora.conv_fwd(x, wo, cfg["bias"][oc:oc + 1], attn=ora.ATTN_MAGNITUDE, k=cfg["k"])
        dy = grad_values(yk.shape[0], SEED_BASE + 99)
        *_, kept_pairs = ora.conv_bwd(x, wo, yk, dy, return_pairs=True)
        dt = time.perf_counter() - t0
        # bwd MACs: 2 x pairs landing on kept outputs (same definition as our arm)
        return macs + 2 * kept_pairs, dt, yk

    for i in range(args.warmup):
        one(i % C_OUT)
    tot_macs, tot_t = 0.0, 0.0
    for i in range(args.steps):
        macs, dt, _ = one(i % C_OUT)
        tot_macs += macs
        tot_t += dt
    value = tot_macs / tot_t / 1e9
    res = {"impl": "reference", "metric": "sparse conv fwd+bwd effective GMAC/s (C4 128^3, rho_up 5%)",
           "value": round(value, 4), "unit": "GMAC/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(tot_t / args.steps * 1e3, 2), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": f"synthetic ({args.values} values, uniform positions, seeded)",
           "config": {"workload": f"C4 sample: one (b, oc) pair of 3D {RES}^3, {C_IN}->1 ch, 3x3x3, rho_f {RHO_F}, "
                                  f"rho_d {args.density}, k={K_SEL}, fwd+bwd", "density": args.density},
           "cpu_baseline": {"value": round(value, 4), "unit": "GMAC/s", "cores": 1, "kind": "oracle",
                            "sample": "one (b, oc) pair of the C4 batch per step, fwd+bwd"},
           "e2e": {"value": round(value, 4), "unit": "GMAC/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)
    return res


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--density", type=float, default=0.02)
    ap.add_argument("--values", default="continuous", choices=["continuous", "dyadic"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--variant", default="measure", choices=["auto", "scatter", "gemm", "measure"],
                    help="forward accumulate variant (SURVEY §8 a3); 'measure' times both once and keeps the faster")
    ap.add_argument("--samples-per-pass", type=int, default=None,
                    help="bounded-memory forward (sparse_conv_fwd_pass, SURVEY §8 f2): samples per pass")
    args = ap.parse_args(argv)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py — sparse conv fwd+bwd on B200 (BASELINE.json metric, configs[3] = C4).

Workload (N=1): 3D 128^3 grid, batch 64, 8 -> 8 channels, 3x3x3 filters pruned to 50%
(rho_f = 0.5), input density rho_d per (b, c) (default 2%; --density), attention with
rho_up = 5% (k = floor(0.05 * 128^3) = 104857 per (b, oc), magnitude variant). One step =
sparse_conv_fwd (Alg. 1 with attention) + sparse_conv_bwd_f64 (Alg. 2: dx and the fp64 dw /
dbias partials) + the SUM all-reduce of dw||dbias across ranks (NCCL, N > 1) and its single
rounding. The all-reduce of step i runs on a side stream and overlaps step i+1's forward (its
rounding is enqueued after that forward). With N GPUs the global batch of 64 is sharded
(strong scaling, BASELINE "batch 64 sharded on 1/2/4/8 GPUs"); `--gpus N` launched as one
process re-executes itself under torch.distributed.run with N ranks (NCCL, NCCL_DEBUG=INFO).
The headline line is rho_d = 2 %; `density_sweep` adds the north-star range 1 % and 5 %.

Metric: effective GMAC/s = algorithmic MACs / time, where fwd MACs are the in-bounds
(input, weight) pairs (Eq. (1) first term) and bwd MACs are 2 x the pairs landing on
kept outputs (dx and dw). HBM GB/s is reported alongside from compulsory bytes.

  python bench.py [--gpus N --steps K --warmup W] [--density 0.02] [--sweep 0.01,0.05] [--impl reference]
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

from synth import (uniform_map, sparse_filter, bias_vector, grad_values, select_samples, surface_occupancy,  # noqa: E402
                   SEED_BASE)

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
class Step:
    """One training step of the C4 layer on this rank's shard: forward (attention), backward with
    the fp64 dw / dbias partials, the all-reduce of step i started on a side stream and finished
    (waited + rounded) after step i+1's forward has been enqueued; two partial buffers alternate."""

    def __init__(self, torch, spc, X, W, bias_t, k, variant, spp, world, dy_t):
        self.torch, self.spc = torch, spc
        self.fwd = spc.FwdPlan(X, W, "magnitude", k, variant, bias_t, spp)
        self.resolved = self.fwd.resolved
        self.cap = self.fwd.capacity
        Y0 = self.fwd(X, W, bias_t)
        self.bwd = spc.BwdPlan(X, W, Y0)
        self.dx = torch.empty(max(X.nnz_bound, 1), device="cuda")
        self.dw = torch.empty(W.keys.numel(), device="cuda")
        self.db = torch.empty(C_OUT, device="cuda")
        side = torch.cuda.Stream() if world > 1 else None
        self.ar = [spc.dp.GradAllReduce(W.keys.numel(), C_OUT, "cuda", stream=side) for _ in range(2)]
        self.i = 0
        self.pending = None
        self.dy = dy_t

    def __call__(self, X, W, bias_t, dy=None):
        Y = self.fwd(X, W, bias_t)
        if self.pending is not None:           # previous step's all-reduce overlapped this forward
            self.pending.finish(self.dw, self.db)
        ar = self.ar[self.i & 1]
        self.bwd.f64(X, W, Y, self.dy if dy is None else dy, self.dx, ar.dw64, ar.db64)
        ar.start()
        self.pending = ar
        self.i += 1
        return Y

    def drain(self):
        if self.pending is not None:
            self.pending.finish(self.dw, self.db)
            self.pending = None


def measure(args, torch, spc, density, rank, world, local, steps, warmup, clocks=True, key_bits=64):
    """Inputs of this rank's shard at `density`, warm-up, the algorithmic work of one step, then
    `steps` timed steps (CUDA events per step on the launching stream; a 512 MB write flushes L2
    between steps, outside the timed intervals)."""
    import torch.distributed as dist

    B_local = BATCH // world
    b0 = rank * B_local
    V = RES ** 3
    cfg = c4_inputs(density, args.values, batch=B_local, b0=b0)
    x, w, bias, k = cfg["x"], cfg["w"], cfg["bias"], cfg["k"]
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims, key_bits=key_bits)
    W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
    bias_t = torch.from_numpy(bias).cuda()
    probe = spc.FwdPlan(X, W, "magnitude", k, args.variant, bias_t, args.samples_per_pass)
    variant = probe.resolved
    cap = probe.capacity
    del probe
    dy_t = torch.from_numpy(grad_values(cap, SEED_BASE + 7 + rank)).cuda()
    step = Step(torch, spc, X, W, bias_t, k, variant, args.samples_per_pass, world, dy_t)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # 512 MB > L2

    for _ in range(warmup):
        step(X, W, bias_t)
    step.drain()
    torch.cuda.synchronize()
    # algorithmic work of one step (measurement plumbing, outside the timed region)
    Y = step(X, W, bias_t)
    step.drain()
    torch.cuda.synchronize()
    ny = int(Y.nnz_dev.item())
    fwd_macs, bwd_macs = algorithmic_macs(torch, X, W, Y.keys[:ny], B_local, V)
    nnz_x, nnz_w = x.nnz, w.nnz
    fwd_bytes = 12 * nnz_x + 12 * nnz_w + 4 * C_OUT + 12 * ny
    bwd_bytes = 12 * nnz_x + 4 * nnz_x + 12 * ny + 16 * nnz_w
    launches0 = spc.kernel_launches()
    step(X, W, bias_t)
    step.drain()
    torch.cuda.synchronize()
    launches_per_step = spc.kernel_launches() - launches0

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local) if clocks else None
    if clk:
        clk.__enter__()
    for i in range(steps):
        flush.zero_()
        evs[i][0].record()
        step(X, W, bias_t)
        if i == steps - 1:
            step.drain()                         # the last all-reduce + rounding belong to the run
        evs[i][1].record()
    torch.cuda.synchronize()
    if clk:
        clk.__exit__()
    if world > 1:
        dist.barrier()
    per_step = [a.elapsed_time(b) for a, b in evs]
    t_ms = float(sum(per_step))
    if world > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
        tot = torch.tensor([fwd_macs + bwd_macs, fwd_bytes + bwd_bytes, fwd_macs, bwd_macs, ny, nnz_x],
                           dtype=torch.float64, device="cuda")
        dist.all_reduce(tot)
        macs_all, bytes_all = float(tot[0].item()), float(tot[1].item())
    else:
        macs_all, bytes_all = float(fwd_macs + bwd_macs), float(fwd_bytes + bwd_bytes)
    ms_per_step = t_ms / steps
    return dict(cfg=cfg, x=x, w=w, X=X, W=W, key_bits=key_bits, bias_t=bias_t, k=k, Y=Y, step=step, flush=flush, variant=variant,
                cap=cap, dy_t=dy_t, B_local=B_local, fwd_macs=fwd_macs, bwd_macs=bwd_macs, ny=ny, nnz_x=nnz_x,
                nnz_w=nnz_w, fwd_bytes=fwd_bytes, bwd_bytes=bwd_bytes, macs_all=macs_all, bytes_all=bytes_all,
                ms_per_step=ms_per_step, per_step=per_step, launches_per_step=launches_per_step,
                clocks=clk.summary() if clk else None,
                value=macs_all / (ms_per_step * 1e-3) / 1e9, hbm_gbs=bytes_all / (ms_per_step * 1e-3) / 1e9)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1801_10585_b200 as spc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spc.load()
    assert BATCH % world == 0
    m = measure(args, torch, spc, args.density, rank, world, local, args.steps, args.warmup)
    args.resolved_variant = m["variant"]

    # ---- per-kernel durations (CUDA events the library records on its stream)
    step, X, W, bias_t = m["step"], m["X"], m["W"], m["bias_t"]
    spc.profile_reset()
    spc.profile_enable(True)
    nprof = max(1, min(3, args.steps))
    for _ in range(nprof):
        m["flush"].zero_()
        step(X, W, bias_t)
        step.drain()
    torch.cuda.synchronize()
    prof = spc.profile_read()
    spc.profile_enable(False)
    phases = {k2: {"ms_per_step": v[0] / nprof, "launches_per_step": v[1] / nprof} for k2, v in prof.items()}
    step_sum = sum(p["ms_per_step"] for p in phases.values()) or 1.0
    top = max(phases, key=lambda n: phases[n]["ms_per_step"])
    pk, src = peaks()
    roof = roofline_for(top, phases[top], m, pk, src)
    roof["share_of_step"] = round(phases[top]["ms_per_step"] / step_sum, 4)
    kernel_roofs = {n: roofline_for(n, phases[n], m, pk, src) for n in ("conv_fwd", "conv_bwd", "fwd_write", "row_index")
                    if n in phases}

    # ---- end to end through the C-ABI with host buffers (pinned), copies inside the region
    e2e = run_e2e(torch, spc, m, args, world, dist if world > 1 else None)

    # ---- the north-star density range (1 % / 5 %) in the same run
    sweep = []
    for d in args.sweep:
        if abs(d - args.density) < 1e-12:
            continue
        md = measure(args, torch, spc, d, rank, world, local, max(1, args.steps // 2), min(args.warmup, 3),
                     clocks=False)
        sweep.append({"density": d, "value": round(md["value"], 3), "unit": "GMAC/s",
                      "ms_per_step": round(md["ms_per_step"], 4), "hbm_gbs": round(md["hbm_gbs"], 2),
                      "hbm_frac_of_peak": round(md["hbm_gbs"] / float(pk.get("hbm_gbs", 6650.0)), 4),
                      "work_per_step": {"fwd_macs": md["fwd_macs"], "bwd_macs": md["bwd_macs"], "nnz_x": md["nnz_x"],
                                        "nnz_y": md["ny"], "compulsory_bytes": md["fwd_bytes"] + md["bwd_bytes"]},
                      "steps": max(1, args.steps // 2)})
        del md
        torch.cuda.empty_cache()

    # ---- the same step with 32-bit key storage (Table 1 "Sparse 32"): device and end to end
    k32 = None
    if not args.no_key32:
        mk = measure(args, torch, spc, args.density, rank, world, local, max(1, args.steps // 2), min(args.warmup, 3),
                     clocks=False, key_bits=32)
        ek = run_e2e(torch, spc, mk, args, world, dist if world > 1 else None)
        k32 = {"key_bits": 32, "value": round(mk["value"], 3), "unit": "GMAC/s", "ms_per_step": round(mk["ms_per_step"], 4),
               "e2e": {"value": round(mk["macs_all"] / (ek["ms_per_step"] * 1e-3) / 1e9, 3), "unit": "GMAC/s",
                       "h2d_bytes_per_step": ek["h2d"], "d2h_bytes_per_step": ek["d2h"],
                       "ms_per_step": round(ek["ms_per_step"], 4)},
               "note": "uint32 keys in and out (valid: 64*8*128^3 = 2^30 keys < 2^32); same work, 4 B less per entry"}
        del mk
        torch.cuda.empty_cache()

    result = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline(m["cfg"], args.cpu_samples)
        e2e_value = (m["macs_all"] / (e2e["ms_per_step"] * 1e-3) / 1e9) if e2e else None
        result = {
            "metric": "sparse conv fwd+bwd effective GMAC/s (C4 128^3, rho_up 5%)",
            "value": round(m["value"], 3),
            "unit": "GMAC/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(m["ms_per_step"], 4),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": f"synthetic ({args.values} values, uniform positions, seeded)",
            "config": {
                "workload": f"C4: 3D {RES}^3, batch {BATCH} (sharded {m['B_local']}/GPU), {C_IN}->{C_OUT} ch, 3x3x3, "
                            f"rho_f {RHO_F}, rho_d {args.density}, rho_up {RHO_UP} (k={K_SEL}), magnitude attention, "
                            f"fwd + bwd(dx,dw,dbias) + dw||dbias all-reduce",
                "global_batch": BATCH,
                "density": args.density,
                "fwd_variant": f"{args.variant} -> {args.resolved_variant}",
                "fwd_samples_per_pass": args.samples_per_pass or "all",
                "fwd_workspace_gb": round(step.fwd.ws_bytes / 1e9, 3),
                "parallelism": f"dp{world}",
                "l2": "flushed between timed steps (512 MB write); inputs also exceed L2",
            },
            "hbm_gbs": round(m["hbm_gbs"], 2),
            "hbm_frac_of_peak": round(m["hbm_gbs"] / float(pk.get("hbm_gbs", 6650.0)), 4),
            "work_per_step": {"fwd_macs": m["fwd_macs"], "bwd_macs": m["bwd_macs"], "nnz_x": m["nnz_x"],
                              "nnz_w": m["nnz_w"], "nnz_y": m["ny"],
                              "compulsory_bytes": m["fwd_bytes"] + m["bwd_bytes"],
                              "fwd_bytes": m["fwd_bytes"], "bwd_bytes": m["bwd_bytes"]},
            "per_step_ms": [round(t, 4) for t in m["per_step"]],
            "kernels": {n: {"ms": round(p["ms_per_step"], 4), "n": p["launches_per_step"],
                            "share": round(p["ms_per_step"] / step_sum, 4)} for n, p in
                        sorted(phases.items(), key=lambda kv: -kv[1]["ms_per_step"])},
            "roofline": roof,
            "kernel_rooflines": kernel_roofs,
            "density_sweep": sweep,
            "key_bits_32": k32,
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 3) if e2e_value else None, "unit": "GMAC/s",
                    "h2d_bytes_per_step": e2e["h2d"], "d2h_bytes_per_step": e2e["d2h"],
                    "ms_per_step": round(e2e["ms_per_step"], 4)} if e2e else None,
            "gpu_launches": int(m["launches_per_step"] * args.steps),
            "gpu_launches_per_step": int(m["launches_per_step"]),
            "clocks": m["clocks"],
        }
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


# Algorithmic bytes per launch (SURVEY §8(d) "Algorithmic bytes per unit of work", 64-bit keys):
# the forward's kernels are charged the whole forward's compulsory traffic (12 B per input, 12 B
# per weight, 4 B per bias, 12 B per output), the backward's the backward's.
def roofline_for(name, ph, m, pk, src):
    t = ph["ms_per_step"] * 1e-3
    hbm = float(pk.get("hbm_gbs", 6650.0))
    sm_mhz = float(pk.get("sm_max_mhz", 1965.0))
    nrows = m["B_local"] * C_IN * RES * RES
    per = {
        "conv_fwd": (m["fwd_bytes"], "fwd: 12 B/input + 12 B/weight + 4 B/bias + 12 B/output (SURVEY 8d)"),
        "conv_bwd": (m["bwd_bytes"], "bwd: 12 B/input + 4 B/dx + 12 B/kept output + 16 B/weight (SURVEY 8d)"),
        "fwd_write": (12 * m["ny"], "12 B per kept output written"),
        "row_index": (8 * m["nnz_x"] + 4 * (nrows + 1), "8 B per key read + 4 B per row pointer"),
    }.get(name)
    if per is None:
        return {"kernel": name, "bound": "unknown", "achieved": None, "peak": None, "unit": None, "frac": None,
                "traffic": None}
    nbytes, what = per
    gbs = nbytes / t / 1e9
    out = {"kernel": name, "bound": "hbm", "achieved": round(gbs, 1), "unit": "GB/s", "peak": hbm,
           "frac": round(gbs / hbm, 4), "traffic": ncu_traffic(name),
           "peak_source": f"{src} (MEASURED_PEAKS.json hbm_gbs)",
           "algorithmic": f"{nbytes} bytes per launch ({what}), {ph['launches_per_step']:g} launch(es) per step",
           "ms": round(ph["ms_per_step"], 4)}
    if name in ("conv_fwd", "conv_bwd"):
        macs = m["fwd_macs"] if name == "conv_fwd" else m["bwd_macs"]
        ffma = 148 * 128 * sm_mhz * 1e6 / 1e12   # TMAC/s: 148 SM x 128 FP32 lanes x clock
        out["alu"] = {"achieved_tmacs": round(macs / t / 1e12, 4), "ffma_peak_tmacs": round(ffma, 2),
                      "frac": round(macs / t / 1e12 / ffma, 4),
                      "note": "secondary: Eq. (1) MACs over the FP32 FMA peak (derived from unit counts)"}
        sp = ncu_shared(name)
        if sp:
            sp["floor_wavefronts"] = int(2 * macs / 32)   # 2 words per MAC (read-modify-write), 32 per wavefront
            out["shared_pipe"] = sp
    return out


def ncu_shared(kernel):
    """The binding resource of the scatter kernels: shared-memory wavefronts per launch and the
    pipe's busy share (ncu, newest committed capture), and the algorithmic floor of the
    read-modify-write scatter (2 words per MAC, 32 words per wavefront). Secondary to `frac`."""
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_traffic.json")), reverse=True):
        try:
            d = json.load(open(path))
        except Exception:
            continue
        if kernel in d and "shared_wavefronts" in d[kernel]:
            e = d[kernel]
            return {"wavefronts": e["shared_wavefronts"], "bank_conflict_wavefronts": e.get("shared_bank_conflicts"),
                    "pct_of_peak": e.get("shared_pipe_pct_of_peak"),
                    "source": os.path.relpath(path, ROOT) + ":" + e["report"],
                    "note": "secondary: the shared-memory pipe the scatter is bound by (ncu --set full)"}
    return None


_NCU_NAME = {"fwd_write": "stream_write", "fwd_resolve": "stream_resolve"}   # library phase -> ncu kernel


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the newest committed ncu --set full capture, or None."""
    kernel = _NCU_NAME.get(kernel, kernel)
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "ncu_traffic.json")), reverse=True):
        try:
            d = json.load(open(path))
        except Exception:
            continue
        if kernel in d:
            return {"bytes": d[kernel]["traffic"], "source": os.path.relpath(path, ROOT) + ":" + d[kernel]["report"]}
    return None


def run_e2e(torch, spc, m, args, world, dist):
    """Same step through the public API with HOST inputs: every step's inputs (x keys/values, dy)
    are copied H2D from pinned memory inside the timed region and its result (dw, dbias, output
    nnz) is read back D2H. Like a data loader, the upload of step i+1 runs on a copy stream into
    the second of two device input buffers while step i computes (the buffer is reused only after
    the step that read it has finished)."""
    x, w, k, bias_t = m["x"], m["w"], m["k"], m["bias_t"]
    kb = m.get("key_bits", 64)
    hk = torch.from_numpy(x.keys.astype(np.uint32).view(np.int32) if kb == 32 else x.keys.view(np.int64)).pin_memory()
    hv = torch.from_numpy(x.values).pin_memory()
    hdy = m["dy_t"].cpu().pin_memory()
    bufs = [(torch.empty_like(hk, device="cuda"), torch.empty_like(hv, device="cuda"),
             torch.empty_like(hdy, device="cuda")) for _ in range(2)]
    W = m["W"]
    Xs = [spc.SparseMap(bk, bv, x.batch, x.channels, x.dims, x.nnz, None) for bk, bv, _ in bufs]
    for bk, bv, bd in bufs:
        bk.copy_(hk)
        bv.copy_(hv)
        bd.copy_(hdy)
    step = Step(torch, spc, Xs[0], W, bias_t, k, args.resolved_variant, args.samples_per_pass, world, bufs[0][2])
    out_dw = torch.empty(W.keys.numel()).pin_memory()
    out_db = torch.empty(C_OUT).pin_memory()
    out_n = torch.empty(1, dtype=torch.int64).pin_memory()
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

    def one(i, last):
        j = i % 2
        if not last:
            upload(i + 1)
        comp.wait_event(loaded[j])
        Y = step(Xs[j], W, bias_t, bufs[j][2])
        consumed[j].record(comp)
        if last:
            step.drain()
        out_dw.copy_(step.dw, non_blocking=True)
        out_db.copy_(step.db, non_blocking=True)
        out_n.copy_(Y.nnz_dev, non_blocking=True)

    def run(n):
        for e in consumed:
            e.record(comp)
        upload(0)
        for i in range(n):
            one(i, i == n - 1)

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
    return {"ms_per_step": ms, "h2d": int(hk.numel() * hk.element_size() + hv.numel() * 4 + hdy.numel() * 4),
            "d2h": int(out_dw.numel() * 4 + out_db.numel() * 4 + 8)}


# --------------------------------------------------------------------- CPU baseline
def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


_CPU_CFG = None   # (x, w, bias, k) inherited by the forked oracle workers (no pickling of the map)


def _oracle_sample(b):
    """fwd+bwd of sample b by the oracle (one worker process of the all-cores leg)."""
    import oracle as ora

    x, w, bias, k = _CPU_CFG
    xs = select_samples(x, [b])
    t0 = time.perf_counter()
    yk, _, _, macs = ora.conv_fwd(xs, w, bias, attn=ora.ATTN_MAGNITUDE, k=k)
    dy = grad_values(yk.shape[0], SEED_BASE + 99 + b)
    *_, kept_pairs = ora.conv_bwd(xs, w, yk, dy, return_pairs=True)
    return macs + 2 * kept_pairs, time.perf_counter() - t0


def cpu_baseline(cfg, nsamples):
    """The oracle (oracle/, plain C, fp64, single-threaded code) on a bounded sample of the same
    workload: one sample on 1 core, then `nsamples` samples on all the host's cores (one forked
    worker process per sample). Reported baseline only."""
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    global _CPU_CFG
    _CPU_CFG = (cfg["x"], cfg["w"], cfg["bias"], cfg["k"])
    macs1, dt1 = _oracle_sample(0)
    ncpu = os.cpu_count() or 1
    ns = max(1, min(nsamples, cfg["x"].batch))
    nw = min(ncpu, ns)
    t0 = time.perf_counter()
    with ProcessPoolExecutor(max_workers=nw, mp_context=mp.get_context("fork")) as ex:
        res = list(ex.map(_oracle_sample, range(ns)))
    dtn = time.perf_counter() - t0
    macsn = sum(r[0] for r in res)
    return {"value": round(macsn / dtn / 1e9, 4), "unit": "GMAC/s", "cores": nw, "kind": "oracle",
            "sample": f"{ns} of {BATCH} samples, fwd+bwd, one worker process per sample on {nw} of {ncpu} cores, "
                      f"{dtn:.1f} s wall",
            "cpu_model": _cpu_model(), "nproc": ncpu,
            "single_core": {"value": round(macs1 / dt1 / 1e9, 4), "unit": "GMAC/s", "cores": 1,
                            "sample": f"1 of {BATCH} samples (b=0), fwd+bwd, {dt1:.1f} s"}}


# ------------------------------------------------------------------- reference arm
def run_reference(args):
    """--impl reference: the oracle as it stands, on this host's cores, on the same config and
    metric. Each step = fwd+bwd of a bounded sample of the C4 batch: one sample per host core, one
    forked worker process per sample (the oracle itself is single-threaded C); the step's time is
    the wall time of that parallel map."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    global _CPU_CFG
    ncpu = os.cpu_count() or 1
    nw = max(1, min(ncpu, BATCH))
    cfg = c4_inputs(args.density, args.values, batch=nw)   # samples 0..nw-1 of the seeded batch
    _CPU_CFG = (cfg["x"], cfg["w"], cfg["bias"], cfg["k"])
    tot_macs, tot_t = 0.0, 0.0
    with ProcessPoolExecutor(max_workers=nw, mp_context=mp.get_context("fork")) as ex:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            res = list(ex.map(_oracle_sample, range(nw)))
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                tot_macs += sum(r[0] for r in res)
                tot_t += dt
    steps = max(1, args.steps)
    value = tot_macs / tot_t / 1e9 if tot_t > 0 else 0.0
    sample = f"{nw} of {BATCH} samples per step, fwd+bwd, one worker process per sample on {nw} of {ncpu} cores"
    res = {"impl": "reference", "metric": "sparse conv fwd+bwd effective GMAC/s (C4 128^3, rho_up 5%)",
           "value": round(value, 4), "unit": "GMAC/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(tot_t / steps * 1e3, 2), "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": f"synthetic ({args.values} values, uniform positions, seeded)",
           "config": {"workload": f"C4 sample: {nw} samples of 3D {RES}^3 per step, {C_IN}->{C_OUT} ch, 3x3x3, "
                                  f"rho_f {RHO_F}, rho_d {args.density}, k={K_SEL}, fwd+bwd", "density": args.density},
           "cpu_baseline": {"value": round(value, 4), "unit": "GMAC/s", "cores": nw, "kind": "oracle",
                            "sample": sample, "cpu_model": _cpu_model(), "nproc": ncpu},
           "e2e": {"value": round(value, 4), "unit": "GMAC/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)
    return res


def _spawn(args, argv):
    """`--gpus N` started as one process: re-execute under torch.distributed.run with N ranks on
    this node (rendezvous on 127.0.0.1), NCCL with its communicator log."""
    import subprocess
    import socket

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd, env=env)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--density", type=float, default=0.02)
    ap.add_argument("--sweep", type=lambda s: [] if s in ("", "none") else [float(v) for v in s.split(",") if v],
                    default=[0.01, 0.05], help="extra densities measured in the same run (north-star range), 'none'")
    ap.add_argument("--values", default="continuous", choices=["continuous", "dyadic"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-samples", type=int, default=16, help="samples of the all-cores oracle leg")
    ap.add_argument("--no-key32", action="store_true", help="skip the 32-bit-key sub-record")
    ap.add_argument("--variant", default="measure", choices=["auto", "scatter", "gemm", "measure"],
                    help="forward accumulate variant (SURVEY §8 a3); 'measure' times both once and keeps the faster")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank plumbing only, gloo on CPU (tests)")
    ap.add_argument("--config", default="c4", choices=["c4", "c3"],
                    help="c4 = BASELINE configs[3] (headline), c3 = configs[2] (point-cloud two-layer step)")
    ap.add_argument("--samples-per-pass", type=int, default=None,
                    help="bounded-memory forward (sparse_conv_fwd_pass, SURVEY §8 f2): samples per pass")
    args = ap.parse_args(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(_spawn(args, argv))
    if args.impl == "reference":
        return run_reference(args)
    if args.dry_run:
        return run_dry(args)
    if args.config == "c3":
        return run_c3(args)
    return run_ours(args)


# ---------------------------------------------------------------------- C3 (configs[2])
C3_RES, C3_BATCH, C3_OCC = 64, 32, 0.02
C3_K = int(C3_OCC * C3_RES ** 3)          # 5242: reading rho_up = rho_d (P:208 protocol rho = rho_up)


def c3_inputs(batch=C3_BATCH, b0=0):
    x = surface_occupancy(batch, C3_RES, C3_OCC, SEED_BASE * 1000 + 300, b0=b0)
    w1 = sparse_filter(1, 32, (3, 3, 3), 1.0, SEED_BASE + 31)
    w2 = sparse_filter(32, 64, (3, 3, 3), 1.0, SEED_BASE + 32)
    return dict(x=x, w1=w1, w2=w2, b1=bias_vector(32, SEED_BASE + 31), b2=bias_vector(64, SEED_BASE + 32))


def run_c3(args):
    """BASELINE configs[2]: 3D point-cloud occupancy 64^3 at 2 % (binary values), batch 32, conv 1->32
    (attention, k = 5242) -> ReLU -> conv 32->64 (attention), forward + backward (dw / dbias of both
    layers, dx of the second, the ReLU backward scatter) [+ the dw||dbias all-reduce per layer].
    Metric as for C4: (Eq. (1) MACs of both layers + 2 x the pairs on kept outputs) / time."""
    import torch
    import torch.distributed as dist
    import torch.nn.functional as F

    import paper_1801_10585_b200 as spc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {args.gpus}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spc.load()
    assert C3_BATCH % world == 0
    B = C3_BATCH // world
    cfg = c3_inputs(B, rank * B)
    x, w1, w2 = cfg["x"], cfg["w1"], cfg["w2"]
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
    W1 = spc.SparseFilter.from_arrays(w1.keys, w1.values, 1, 32, (3, 3, 3))
    W2 = spc.SparseFilter.from_arrays(w2.keys, w2.values, 32, 64, (3, 3, 3))
    b1, b2 = torch.from_numpy(cfg["b1"]).cuda(), torch.from_numpy(cfg["b2"]).cuda()
    f1 = spc.FwdPlan(X, W1, "magnitude", C3_K, args.variant, b1)
    Y1 = f1(X, W1, b1)
    R1, src1 = spc.sparse_relu(Y1)
    f2 = spc.FwdPlan(R1, W2, "magnitude", C3_K, args.variant, b2)
    Y2 = f2(R1, W2, b2)
    g1, g2 = spc.BwdPlan(X, W1, Y1), spc.BwdPlan(R1, W2, Y2)
    dy2 = torch.from_numpy(grad_values(Y2.nnz_bound, SEED_BASE + 33 + rank)).cuda()
    dR1 = torch.empty(max(R1.nnz_bound, 1), device="cuda")
    side = torch.cuda.Stream() if world > 1 else None
    ar1 = spc.dp.GradAllReduce(w1.nnz, 32, "cuda", stream=side)
    ar2 = spc.dp.GradAllReduce(w2.nnz, 64, "cuda", stream=side)
    dw1, db1 = torch.empty(w1.nnz, device="cuda"), torch.empty(32, device="cuda")
    dw2, db2 = torch.empty(w2.nnz, device="cuda"), torch.empty(64, device="cuda")
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    state = {}

    def step():
        Y1 = f1(X, W1, b1)
        R1, src1 = spc.sparse_relu(Y1)
        Y2 = f2(R1, W2, b2)
        g2.f64(R1, W2, Y2, dy2, dR1, ar2.dw64, ar2.db64)
        ar2.start()                               # layer 2's exchange overlaps layer 1's backward
        dY1 = spc.sparse_scatter_grad(src1, dR1, R1.nnz_bound, Y1.nnz_bound, R1.nnz_dev, sorted=True)
        g1.f64(X, W1, Y1, dY1, None, ar1.dw64, ar1.db64)
        ar1.start()
        ar2.finish(dw2, db2)
        ar1.finish(dw1, db1)
        state.update(Y1=Y1, R1=R1, Y2=Y2)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # algorithmic work (measurement plumbing): Eq. (1) pairs per layer from mask correlations
    V = C3_RES ** 3

    def pairs(inp, ch_in, w, ch_out, ykeys):
        wm = torch.zeros(ch_out * ch_in * 27, device="cuda")
        wm[w.keys.long()] = 1.0
        wm = wm.view(ch_out, ch_in, 3, 3, 3)
        keys = inp.keys[:inp.nnz()]
        fwd, kept = 0, 0
        for s0 in range(0, B, 4):
            nb = min(4, B - s0)
            lo, hi = s0 * ch_in * V, (s0 + nb) * ch_in * V
            m = torch.zeros(nb * ch_in * V, device="cuda")
            m[keys[(keys >= lo) & (keys < hi)] - lo] = 1.0
            cnt = F.conv3d(m.view(nb, ch_in, C3_RES, C3_RES, C3_RES), wm, padding=1)
            fwd += int(cnt.double().sum().item())
            ylo, yhi = s0 * ch_out * V, (s0 + nb) * ch_out * V
            kept += int(cnt.reshape(-1)[ykeys[(ykeys >= ylo) & (ykeys < yhi)] - ylo].double().sum().item())
        return fwd, 2 * kept

    torch.backends.cudnn.allow_tf32 = False
    step()
    torch.cuda.synchronize()
    Y1, R1, Y2 = state["Y1"], state["R1"], state["Y2"]
    fm1, bm1 = pairs(X, 1, W1, 32, Y1.keys[:Y1.nnz()])
    fm2, bm2 = pairs(R1, 32, W2, 64, Y2.keys[:Y2.nnz()])
    macs = fm1 + bm1 + fm2 + bm2
    l0 = spc.kernel_launches()
    step()
    torch.cuda.synchronize()
    lps = spc.kernel_launches() - l0
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record()
            step()
            evs[i][1].record()
        torch.cuda.synchronize()
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    macs_all = float(macs)
    if world > 1:
        t = torch.tensor([t_ms, macs], dtype=torch.float64, device="cuda")
        tmax = t[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:])
        t_ms, macs_all = float(tmax.item()), float(t[1].item())
    ms = t_ms / args.steps
    spc.profile_reset()
    spc.profile_enable(True)
    step()
    torch.cuda.synchronize()
    prof = spc.profile_read()
    spc.profile_enable(False)
    if rank == 0:
        res = {"metric": "sparse conv fwd+bwd effective GMAC/s (C3 64^3 surface 2%, 1->32->64)",
               "value": round(macs_all / (ms * 1e-3) / 1e9, 3), "unit": "GMAC/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f32",
               "data": "synthetic (voxelised sphere shells and plane patches, binary values, seeded)",
               "config": {"workload": f"C3: 3D {C3_RES}^3 occupancy {C3_OCC}, batch {C3_BATCH} (sharded {B}/GPU), "
                                      f"conv 1->32 (attention k={C3_K}) -> ReLU -> conv 32->64 (attention k={C3_K}), "
                                      "3x3x3 dense filters, fwd + bwd + dw||dbias all-reduce per layer",
                          "fwd_variants": f"{args.variant} -> {f1.resolved}, {f2.resolved}",
                          "parallelism": f"dp{world}", "l2": "flushed between timed steps (512 MB write)"},
               "work_per_step": {"fwd_macs_l1": fm1, "bwd_macs_l1": bm1, "fwd_macs_l2": fm2, "bwd_macs_l2": bm2,
                                 "nnz_x": int(x.nnz), "nnz_y1": Y1.nnz(), "nnz_relu": R1.nnz(), "nnz_y2": Y2.nnz()},
               "kernels": {n: round(v[0], 4) for n, v in sorted(prof.items(), key=lambda kv: -kv[1][0])},
               "gpu_launches": int(lps * args.steps), "gpu_launches_per_step": int(lps), "clocks": clk.summary()}
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_dry(args):
    """--dry-run: the multi-rank plumbing of run_ours without a GPU (gloo): rank / world from the
    launcher, the batch shard of each rank, the fp64 SUM all-reduce + single rounding of a
    dw||dbias buffer (dp.GradAllReduce) and the max-over-ranks timing; rank 0 prints one line.
    Covered by tests/test_bench_spawn.py (world size 2 on CPU)."""
    import torch
    import torch.distributed as dist

    from paper_1801_10585_b200 import dp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {args.gpus}")
    if world > 1:
        dist.init_process_group("gloo")
    b0, b1 = dp.shard_range(BATCH, world, rank)
    nw = 864
    ar = dp.GradAllReduce(nw, C_OUT, "cpu")
    ar.dw64.copy_(torch.arange(nw, dtype=torch.float64) * (rank + 1) / 64.0)
    ar.db64.fill_(float(b1 - b0))
    dw, db = torch.empty(nw), torch.empty(C_OUT)
    ar(dw, db)
    want = torch.arange(nw, dtype=torch.float64) * (world * (world + 1) / 2) / 64.0
    t = dp.max_over_ranks(float(rank), "cpu")
    shards = [None] * world
    if world > 1:
        dist.all_gather_object(shards, (b0, b1))
    else:
        shards = [(b0, b1)]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "shards": shards,
                          "allreduce_ok": bool(torch.equal(dw, want.to(torch.float32))) and float(db[0]) == BATCH,
                          "max_over_ranks": t}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

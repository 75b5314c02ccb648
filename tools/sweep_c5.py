"""C5 density sweep (BASELINE.json configs[4], SURVEY §8 d): 64^3 grid, batch 8, 32 -> 32 channels,
dense 3x3x3 filter, densities 0.1% .. 50%. Times, per density, the sparse forward with each
accumulate variant (S scatter, G tensor cores) and the library's per-layer choice, the sparse
backward (dx, dw, dbias), and the dense cuDNN conv3d forward / backward on the densified input
(fp32 with TF32 off, and TF32 on) -- the sparse/dense crossover. CUDA events, warm-up first.

  python tools/sweep_c5.py [--densities 0.001,0.01,...] [--sites indep|shared] [--out file.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import uniform_map, sparse_filter, bias_vector, grad_values, SEED_BASE  # noqa: E402


def timed(torch, fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    import torch

    import paper_1801_10585_b200 as spc

    ap = argparse.ArgumentParser()
    ap.add_argument("--densities", default="0.001,0.002,0.005,0.01,0.02,0.05,0.1,0.2,0.5")
    ap.add_argument("--sites", default="indep", choices=["indep", "shared"])
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--res", type=int, default=64)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    B, R, CI, CO = args.batch, args.res, 32, 32
    V = R ** 3
    w = sparse_filter(CI, CO, (3, 3, 3), 1.0, SEED_BASE + 5)
    bias = bias_vector(CO, SEED_BASE + 5)
    W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
    bias_t = torch.from_numpy(bias).cuda()
    wd = torch.zeros(CO * CI * 27, dtype=torch.float32)
    wd[torch.from_numpy(w.keys.view(np.int64))] = torch.from_numpy(w.values)
    wdense = wd.view(CO, CI, 3, 3, 3).cuda()
    out = open(args.out, "w") if args.out else None
    for d in [float(s) for s in args.densities.split(",")]:
        x = uniform_map(B, CI, (R, R, R), d, SEED_BASE * 1000 + 500 + int(d * 1e4), sites=args.sites)
        X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
        row = {"config": "C5", "density": d, "sites": args.sites, "batch": B, "grid": R, "c_in": CI, "c_out": CO,
               "nnz_x": int(X.nnz_bound)}
        macs = int(X.nnz_bound) * 27 * CO   # upper bound of Eq. (1) pairs (boundary pairs included)
        row["fwd_macs_bound"] = macs
        for attn, k in (("none", 0), ("magnitude", max(1, int(d * V)))):
            for var in ("scatter", "gemm"):
                plan = spc.FwdPlan(X, W, attn, k, var)
                row[f"fwd_{attn}_{var}_ms"] = round(timed(torch, lambda: plan(X, W, bias_t)), 4)
                del plan
            plan = spc.FwdPlan(X, W, attn, k, "measure", bias_t)
            row[f"fwd_{attn}_choice"] = plan.resolved
        # backward of the exact (attn none) layer: dy on every output entry
        Y = spc.FwdPlan(X, W, "magnitude", max(1, int(d * V)), "auto")(X, W, bias_t).exact()
        dy = torch.from_numpy(grad_values(Y.nnz_bound, SEED_BASE + 9)).cuda()
        bwd = spc.BwdPlan(X, W, Y)
        dx = torch.empty(max(X.nnz_bound, 1), device="cuda")
        dw = torch.empty(W.keys.numel(), device="cuda")
        db = torch.empty(CO, device="cuda")
        row["bwd_ms"] = round(timed(torch, lambda: bwd(X, W, Y, dy, dx, dw, db), reps=3, warm=1), 4)
        # dense cuDNN baseline on the densified input
        xd = torch.zeros(B * CI * V, dtype=torch.float32, device="cuda")
        xd[X.keys] = X.values
        xd = xd.view(B, CI, R, R, R).requires_grad_(True)
        wdd = wdense.clone().requires_grad_(True)
        for tf32 in (False, True):
            torch.backends.cudnn.allow_tf32 = tf32
            tag = "tf32" if tf32 else "fp32"
            f = lambda: torch.nn.functional.conv3d(xd, wdd, bias_t, padding=1)
            row[f"cudnn_fwd_{tag}_ms"] = round(timed(torch, f), 4)
            yd = f()
            g = torch.randn_like(yd)
            row[f"cudnn_fwdbwd_{tag}_ms"] = round(
                timed(torch, lambda: torch.autograd.grad(f(), (xd, wdd), g), reps=3), 4)
        torch.backends.cudnn.allow_tf32 = False
        print(json.dumps(row), flush=True)
        if out:
            out.write(json.dumps(row) + "\n")
            out.flush()
        del X, Y, xd, bwd


if __name__ == "__main__":
    main()

"""HBM roofline of the streaming ops: each op of the C-ABI on
a C4-sized map (128^3, batch 64, 8 channels, 5 % density per channel = the forward's output
bound at rho_up = 5 %, 53.7 M entries, 644 MB of keys + values: larger than the 126 MB L2, which
is also flushed between iterations). Inputs are built on the device (timing tool, not a parity
test). Per op: device time of the whole call (CUDA events, median of --iters), the compulsory
HBM bytes (read every input once, write every output once) and their ratio to the measured copy
bandwidth of MEASURED_PEAKS.json.

  python tools/bench_stream_ops.py [--iters 10] [--out profiles/r01/stream_ops.json]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1801_10585_b200 as spc

    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--density", type=float, default=0.05)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    spc.load()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    R, B, C = 128, 64, 8
    V = R ** 3
    g = torch.Generator(device="cuda").manual_seed(1801)
    keys = []
    for s in range(B * C):   # per-(b, c) Bernoulli(density) positions, key order
        p = torch.nonzero(torch.rand(V, device="cuda", generator=g) < args.density).squeeze(1)
        keys.append(p + s * V)
    keys = torch.cat(keys)
    n = keys.numel()
    vals = torch.randn(n, device="cuda", generator=g)
    X = spc.SparseMap(keys, vals, B, C, (R, R, R), n, None)
    flush = torch.empty(512 * 2 ** 20 // 4, device="cuda")

    def timed(fn):
        ts = []
        out = None
        for i in range(args.iters + 2):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = fn()
            b.record()
            b.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b))
        return statistics.median(ts), out

    rows = []

    last = {}

    def timed_phases(fn):
        # one more call with the library's per-phase CUDA-event brackets (outside the timed runs)
        spc.profile_reset()
        spc.profile_enable(True)
        fn()
        torch.cuda.synchronize()
        spc.profile_enable(False)
        return {k2: round(v[0], 4) for k2, v in spc.profile_read().items()}

    def report(name, ms, nbytes, note, fn=None):
        gbs = nbytes / (ms * 1e-3) / 1e9
        rows.append({"op": name, "ms": round(ms, 4), "bytes": int(nbytes), "gbs": round(gbs, 1),
                     "frac_of_hbm": round(gbs / peak, 3), "bytes_counted": note,
                     "phases_ms": timed_phases(fn) if fn else None})
        print(f"{name:28s} {ms:8.4f} ms {nbytes / 1e9:7.3f} GB {gbs:8.1f} GB/s  {gbs / peak * 100:5.1f} %")

    from bench import ClockSampler

    clk = ClockSampler(0).__enter__()   # SM clock + throttle reasons during all timed runs
    ms, (y, src) = timed(lambda: spc.sparse_relu(X))
    nk = y.nnz()
    report("sparse_relu", ms, 12 * n + 20 * nk, "keys+values read; kept keys+values+src written",
           lambda: spc.sparse_relu(X))
    ms, (p, arg) = timed(lambda: spc.sparse_maxpool(X, (2, 2, 2)))
    npool = p.nnz()
    report("sparse_maxpool 2x2x2", ms, 12 * n + 20 * npool, "keys+values read; pooled keys+values+argmax written",
           lambda: spc.sparse_maxpool(X, (2, 2, 2)))
    kk = int(0.025 * V)
    ms, (t, tsrc) = timed(lambda: spc.attention_topk(X, "magnitude", kk))
    nt = t.nnz()
    report(f"attention_topk k={kk}", ms, 12 * n + 20 * nt, "keys+values read; kept keys+values+src written",
           lambda: spc.attention_topk(X, "magnitude", kk))
    n1 = int(torch.searchsorted(keys, torch.tensor([C * V], device="cuda")).item())   # sample 0 only
    one = spc.SparseMap(keys[:n1], vals[:n1], 1, C, (R, R, R), n1, None)
    ms, (t1, _) = timed(lambda: spc.attention_topk(one, "magnitude", kk))
    report(f"attention_topk k={kk}, 1 sample (8 segments)", ms, 12 * n1 + 20 * t1.nnz(),
           "keys+values read; kept keys+values+src written", lambda: spc.attention_topk(one, "magnitude", kk))
    dy = torch.randn(max(nk, 1), device="cuda", generator=g)
    ms, _ = timed(lambda: spc.sparse_scatter_grad(src, dy, nk, n))
    report("sparse_scatter_grad (relu)", ms, 12 * nk + 4 * n, "src+dy read; dx written (zeros included)")
    ms, _ = timed(lambda: spc.sparse_scatter_grad(src, dy, nk, n, sorted=True))
    report("sparse_scatter_grad_sorted (relu)", ms, 12 * nk + 4 * n, "src+dy read; dx written once (zeros included)")
    ms, k32 = timed(lambda: spc.keys_narrow(X))
    report("keys_narrow", ms, 12 * n, "8 B read + 4 B written per key")
    ms, _ = timed(lambda: spc.keys_widen(k32, n))
    report("keys_widen", ms, 12 * n, "4 B read + 8 B written per key")
    n8 = int(torch.searchsorted(keys, torch.tensor([(B // 8) * C * V], device="cuda")).item())   # samples 0..7
    half = spc.SparseMap(keys[:n8], vals[:n8], B // 8, C, (R, R, R), n8, None)
    ms, _ = timed(lambda: spc.sparse_to_dense(half))
    report("sparse_to_dense (8 samples)", ms, 12 * n8 + 4 * (B // 8) * C * V, "keys+values read; dense written")
    clk.__exit__()
    res = {"workload": f"{R}^3 x batch {B} x {C} ch, density {args.density} per channel, {n} entries, randn values",
           "peak_hbm_gbs": peak, "iters": args.iters, "l2": "512 MB flush between iterations", "ops": rows,
           "clocks": clk.summary()}
    print(json.dumps(res))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

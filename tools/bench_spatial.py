"""Spatial sharding (f4) measured on one GPU with virtual shards: one C4-setting sample (8 -> 8
channels, 3x3x3, rho_f 0.5, rho_d 2 %, k = 5 % of the grid, magnitude attention) on an R^3 grid,
forward + backward on one GPU, then split into G = 2 / 4 / 8 plane ranges (spatial.SpatialConv
with LoopbackComm). Per G: the GPU time each rank's own work takes (CUDA events around every
rank's kernels; the ranks run one after the other on this GPU), the max over ranks (what a step
would cost per GPU, communication excluded), the halo bytes a rank sends, the all-reduce volume,
and a parity check against the single-GPU layer (kept keys identical, values / dx / dw equal).

python tools/bench_spatial.py [--res 256] [--reps 3] [--out profiles/r02/spatial_r02e.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--res", type=int, default=256)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import numpy as np
    import torch

    import paper_1801_10585_b200 as spc
    from paper_1801_10585_b200.spatial import LoopbackComm, SpatialConv, extract_planes
    from synth import uniform_map, sparse_filter, bias_vector, grad_values
    from bench import ClockSampler

    spc.load()
    torch.cuda.set_device(0)
    R = args.res
    dims = (R, R, R)
    V = R ** 3
    k = int(0.05 * V)
    t0 = time.time()
    x = uniform_map(1, 8, dims, 0.02, 8800, values="continuous")
    w = sparse_filter(8, 8, (3, 3, 3), 0.5, 8801, values="continuous")
    bias = bias_vector(8, 8802, values="continuous")
    X = spc.SparseMap.from_arrays(x.keys, x.values, 1, 8, dims)
    Wf = spc.SparseFilter.from_arrays(w.keys, w.values, 8, 8, (3, 3, 3))
    bt = torch.from_numpy(bias).cuda()
    gen_s = time.time() - t0

    def single():
        Y = spc.sparse_conv_fwd(X, Wf, bt, "magnitude", k).exact()
        return Y

    Y = single()
    dy = torch.from_numpy(grad_values(Y.nnz_bound, 8803, values="continuous")).cuda()
    dX, dW, dB = spc.sparse_conv_bwd(X, Wf, Y, dy)
    clk = ClockSampler(0).__enter__()
    ms1 = []
    for _ in range(args.reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        Yr = single()
        spc.sparse_conv_bwd(X, Wf, Yr, dy)
        b.record()
        torch.cuda.synchronize()
        ms1.append(a.elapsed_time(b))
    spc.profile_reset()
    spc.profile_enable(True)
    Yp = single()
    spc.sparse_conv_bwd(X, Wf, Yp, dy)
    torch.cuda.synchronize()
    prof1 = sorted(spc.profile_read().items(), key=lambda kv: -kv[1][0])
    spc.profile_enable(False)
    res = {"workload": f"one sample {R}^3, 8->8 ch, 3x3x3, rho_f 0.5, rho_d 0.02, k = 5% of V "
                       "(magnitude attention), fwd + bwd (dx, dw, dbias)",
           "inputs": int(X.nnz_bound), "kept_outputs": int(Y.nnz_bound), "gen_s": round(gen_s, 1),
           "single_gpu_ms": round(min(ms1), 3),
           "single_phases_ms": {n: round(v[0], 3) for n, v in prof1[:12]}, "shards": []}
    for G in [int(g) for g in args.worlds.split(",")]:
        layer = SpatialConv(LoopbackComm(G), R, timing=True)
        rng = layer.ranges()
        xs = [extract_planes(X, a, e)[0].exact() for a, e in rng]
        dys = []
        for (a, e) in rng:
            ry, yi = extract_planes(Y, a, e, src_index=True)
            dys.append(dy[yi[:ry.exact().nnz_bound]].contiguous())
        per = []
        for rep in range(args.reps + 1):
            layer.halo_bytes = [0] * G
            layer.rank_ms()
            ys = [y.exact() for y in layer.forward(xs, Wf, bt, "magnitude", k)]
            outs = layer.backward(xs, Wf, ys, dys)
            ms = layer.rank_ms()
            if rep:
                per.append(ms)
        best = min(per, key=max)
        halo = list(layer.halo_bytes)
        spc.profile_reset()
        spc.profile_enable(True)
        ys = [y.exact() for y in layer.forward(xs, Wf, bt, "magnitude", k)]
        outs = layer.backward(xs, Wf, ys, dys)
        torch.cuda.synchronize()
        prof = sorted(spc.profile_read().items(), key=lambda kv: -kv[1][0])
        spc.profile_enable(False)
        ok_keys = all(torch.equal(y.keys, extract_planes(Y, a, e)[0].exact().keys) for y, (a, e) in zip(ys, rng))
        vals_err = max(float((y.values - extract_planes(Y, a, e)[0].exact().values).abs().max())
                       for y, (a, e) in zip(ys, rng) if y.nnz_bound)
        dx_err = 0.0
        for (dx, _, _), (a, e), xsh in zip(outs, rng, xs):
            _, xi = extract_planes(X, a, e, src_index=True)
            if xsh.nnz_bound:
                dx_err = max(dx_err, float((dx - dX[xi[:xsh.nnz_bound]]).abs().max()))
        dw_err = float((outs[0][1] - dW).abs().max())
        res["shards"].append({
            "G": G, "rank_ms": [round(v, 3) for v in best], "max_rank_ms": round(max(best), 3),
            "speedup_vs_single": round(min(ms1) / max(best), 2),
            "phases_all_ranks_ms": {n: round(v[0], 3) for n, v in prof[:12]},
            "halo_bytes_per_rank_max": max(halo),
            "allreduce_bytes": 8 * (int(Wf.keys.numel()) + 8),
            "select_allreduce_bytes_per_round": 4 * 8 * 256,
            "parity": {"kept_keys_equal": bool(ok_keys), "max_abs_value_diff": vals_err, "max_abs_dx_diff": dx_err,
                       "max_abs_dw_diff": dw_err}})
        print(json.dumps(res["shards"][-1]), flush=True)
    res["clocks"] = clk.summary()
    clk.__exit__(None, None, None)
    line = json.dumps(res)
    print(line)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()

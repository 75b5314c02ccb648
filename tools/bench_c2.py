"""C2 network step (BASELINE.json configs[1], SURVEY §8 d): MNIST-like 28x28 strokes, batch 256,
3 x [sparse conv 3x3 + attention (rho_up 15%, magnitude) -> sparse ReLU -> sparse max-pool 2x2],
channels 1 -> 8 -> 16 -> 32, forward + backward (dx, dw, dbias of every conv; ReLU / pool backward
scatters), synthetic dy on the final pooled map. Every op goes through the C-ABI; layer sizes chain
on the device (output counts are device words), so the whole step has no host synchronisation and
is captured once into a CUDA graph (the config is launch-latency bound: µs-scale kernels).

Reports eager and graph-replayed µs per step (CUDA events), kernels per step, and the Eq. (1) MACs
of the step (counted once on the device, outside the timed region).

  python tools/bench_c2.py [--batch 256] [--steps 50] [--warmup 5]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import mnist_like, sparse_filter, bias_vector, SEED_BASE  # noqa: E402

CHANS = [1, 8, 16, 32]
KSEL = [int(0.15 * 28 * 28), int(0.15 * 14 * 14), int(0.15 * 7 * 7)]   # 117, 29, 7 (reading R5: floor)


def main():
    import torch
    import torch.nn.functional as F

    import paper_1801_10585_b200 as spc

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    spc.load()
    x = mnist_like(args.batch, SEED_BASE + 2)
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
    Ws = [sparse_filter(CHANS[i], CHANS[i + 1], (3, 3), 1.0, SEED_BASE + 20 + i) for i in range(3)]
    Wd = [spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize) for w in Ws]
    Bd = [torch.from_numpy(bias_vector(CHANS[i + 1], SEED_BASE + 30 + i)).cuda() for i in range(3)]
    launches = []

    def step():
        n0 = spc.kernel_launches()
        acts = []
        cur = X
        for i in range(3):
            y = spc.sparse_conv_fwd(cur, Wd[i], Bd[i], "magnitude", KSEL[i], variant="scatter")
            r, rsrc = spc.sparse_relu(y)
            p, parg = spc.sparse_maxpool(r, (2, 2))
            acts.append((cur, y, r, rsrc, p, parg))
            cur = p
        # synthetic dL/dp on the final pooled map (capacity-sized, rows past the count unused)
        dp = torch.ones(cur.nnz_bound, device="cuda") * 0.01
        grads = []
        for i in reversed(range(3)):
            xin, y, r, rsrc, p, parg = acts[i]
            dr = spc.sparse_scatter_grad(parg, dp, p.nnz_bound, r.nnz_bound, p.nnz_dev)
            dyv = spc.sparse_scatter_grad(rsrc, dr, r.nnz_bound, y.nnz_bound, r.nnz_dev, sorted=True)
            dx, dw, db = spc.sparse_conv_bwd(xin, Wd[i], y, dyv, need_dx=i > 0)
            grads.append((dw, db))
            dp = dx
        launches.append(spc.kernel_launches() - n0)
        return acts, grads

    def timed(fn, n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / n * 1e3

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    eager_us = timed(step, args.steps)
    kernels = launches[-1]

    # Eq. (1) MACs of the step: in-bounds (input, weight) pairs per layer (dense correlation of the
    # occupancy masks, exact integers) -- measurement plumbing, outside the timed region
    acts, _ = step()
    torch.cuda.synchronize()
    macs = 0
    for i in range(3):
        xin = acts[i][0]
        n = xin.nnz()
        H, Wd_ = xin.dims
        m = torch.zeros(xin.batch * xin.channels * H * Wd_, device="cuda")
        m[xin.keys[:n]] = 1.0
        wm = torch.zeros(CHANS[i + 1] * CHANS[i] * 9, device="cuda")
        wm[Wd[i].keys] = 1.0
        macs += int(F.conv2d(m.view(xin.batch, xin.channels, H, Wd_), wm.view(CHANS[i + 1], CHANS[i], 3, 3),
                             padding=1).double().sum().item())

    # CUDA graph of the whole step (allocations come from the graph's private pool)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(args.warmup):
        g.replay()
    torch.cuda.synchronize()
    graph_us = timed(g.replay, args.steps)
    # per-phase device time of one eager step (CUDA-event brackets of the library, outside the timing)
    spc.profile_reset()
    spc.profile_enable(True)
    step()
    torch.cuda.synchronize()
    spc.profile_enable(False)
    phases = {k: [round(v[0] * 1e3, 1), v[1]] for k, v in sorted(spc.profile_read().items(), key=lambda kv: -kv[1][0])}
    print(json.dumps({"config": "C2: MNIST-like 28x28, batch %d, 3 x [conv3x3+attn(15%%)->ReLU->pool2], 1-8-16-32, "
                      "fwd+bwd" % args.batch, "eager_us_per_step": round(eager_us, 1),
                      "graph_us_per_step": round(graph_us, 1), "kernels_per_step": kernels,
                      "fwd_macs_per_step": macs, "fwd_gmac_s_graph": round(macs / graph_us / 1e3, 2),
                      "phases_us_eager": phases}))


if __name__ == "__main__":
    main()

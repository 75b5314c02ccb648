"""OctNet3-64^3 sparse trunk (Appendix B Table 2): on synthetic point-cloud
occupancy grids (voxelised sphere shells and planes, ~2 % of 64^3, value 1.0), batch 32:
  conv(1,8) conv(8,8) conv(8,8) pool(2) conv(8,16) conv(16,16) conv(16,16) pool(2)
  conv(16,24) conv(24,24) conv(24,24) sparseToDense()
every conv 3x3x3 with attention (magnitude) at the block's rho (0.06 / 0.14 / 0.33, the §4.3
setting) followed by sparse ReLU; forward and backward (dx, dw, dbias through every layer, the
ReLU / pool scatters and the sparseToDense gather) with a synthetic gradient on the dense output.
The dense head after sparseToDense is outside the sparse hot path and not run. The whole step
chains on device counts and is captured into one CUDA graph.

  python tools/bench_octnet.py [--batch 32] [--steps 20]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from synth import surface_occupancy, sparse_filter, bias_vector, SEED_BASE  # noqa: E402

BLOCKS = [(1, 8, 0.06), (8, 16, 0.14), (16, 24, 0.33)]   # (c_in of the block, c_out, rho_up)


def main():
    import torch

    import paper_1801_10585_b200 as spc

    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--res", type=int, default=64)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--variant", default="measure", choices=["scatter", "gemm", "auto", "measure"])
    args = ap.parse_args()
    spc.load()
    x = surface_occupancy(args.batch, args.res, 0.02, SEED_BASE + 40)
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
    layers = []
    seed = SEED_BASE + 50
    for bi, (ci, co, rho) in enumerate(BLOCKS):
        res = args.res >> bi
        k = max(1, int(rho * res ** 3))
        for li in range(3):
            cin = ci if li == 0 else co
            w = sparse_filter(cin, co, (3, 3, 3), 1.0, seed)
            b = bias_vector(co, seed)
            seed += 1
            layers.append((spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize),
                           torch.from_numpy(b).cuda(), k, li == 2 and bi < 2))
    launches = []

    def step():
        n0 = spc.kernel_launches()
        tape = []
        cur = X
        for W, B, k, pool in layers:
            y = spc.sparse_conv_fwd(cur, W, B, "magnitude", k, variant=args.variant)
            r, rsrc = spc.sparse_relu(y)
            rec = [cur, W, y, r, rsrc, None, None]
            cur = r
            if pool:
                p, parg = spc.sparse_maxpool(r, (2, 2, 2))
                rec[5], rec[6] = p, parg
                cur = p
            tape.append(rec)
        dense = spc.sparse_to_dense(cur)
        g = torch.full_like(dense, 1e-3)
        dcur = spc.sparse_to_dense_bwd(cur, g)
        for xin, W, y, r, rsrc, p, parg in reversed(tape):
            if p is not None:
                dcur = spc.sparse_scatter_grad(parg, dcur, p.nnz_bound, r.nnz_bound, p.nnz_dev)
            dy = spc.sparse_scatter_grad(rsrc, dcur, r.nnz_bound, y.nnz_bound, r.nnz_dev, sorted=True)
            dx, dw, db = spc.sparse_conv_bwd(xin, W, y, dy, need_dx=xin is not X)
            dcur = dx
        launches.append(spc.kernel_launches() - n0)

    def timed(fn, n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / n

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    eager = timed(step, args.steps)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            step()
    torch.cuda.current_stream().wait_stream(s)
    gph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gph):
        step()
    for _ in range(args.warmup):
        gph.replay()
    torch.cuda.synchronize()
    graph = timed(gph.replay, args.steps)
    # per-phase device time of one eager step (CUDA-event brackets of the library, outside the timing)
    spc.profile_reset()
    spc.profile_enable(True)
    step()
    torch.cuda.synchronize()
    spc.profile_enable(False)
    phases = {k: [round(v[0], 3), v[1]] for k, v in sorted(spc.profile_read().items(), key=lambda kv: -kv[1][0])}
    print(json.dumps({"config": f"OctNet3-{args.res}^3 sparse trunk (Table 2), batch {args.batch}, surface occupancy "
                      f"2%, 9 convs + attention (0.06/0.14/0.33) + ReLU, 2 pools, sparseToDense; fwd+bwd",
                      "eager_ms_per_step": round(eager, 3), "graph_ms_per_step": round(graph, 3),
                      "kernels_per_step": launches[-1], "input_nnz": int(X.nnz_bound), "variant": args.variant,
                      "choices": sorted(set(spc.ops._MEASURED.values())) if args.variant == "measure" else None,
                      "phases_ms_eager": phases}))


if __name__ == "__main__":
    main()

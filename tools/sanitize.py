"""One small invocation of every C-ABI op (forward with the sampled threshold and with the
redo pass, backward, data-parallel backward, ReLU, max-pool, top-k, scatter-grad, rank 4),
for compute-sanitizer (memcheck / racecheck / synccheck / initcheck). Inputs are seeded;
no checks here -- parity is the tests' job. Usage:
  compute-sanitizer --tool racecheck python tools/sanitize.py"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1801_10585_b200 as spc
    from synth import uniform_map, sparse_filter, bias_vector, grad_values

    spc.load()
    cases = [((40, 96, 64), 1, 3, 4, (3, 3, 3), 0.6),        # sampled threshold (>= 8 * P tiles)
             ((9, 7, 11), 2, 3, 5, (3, 3, 3), 0.6),          # small, no sampling
             ((5, 6, 7, 9), 1, 2, 3, (3, 3, 3, 3), 0.6),     # rank 4
             ((28, 28), 2, 1, 8, (3, 3), 0.6),
             ((10, 12, 16), 1, 16, 16, (3, 3, 3), 1.0),      # forward records in global memory
             ((24, 24, 16), 1, 32, 8, (3, 3, 3), 0.6)]       # backward in two passes per item
    for dims, B, ci, co, ks, rho_f in cases:
        x = uniform_map(B, ci, dims, 0.05, 7000, values="dyadic")
        w = sparse_filter(ci, co, ks, rho_f, 7001, values="dyadic")
        bias = torch.from_numpy(bias_vector(co, 7002, values="dyadic")).cuda()
        X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
        W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
        V = 1
        for d in dims:
            V *= d
        k = max(1, V // 20)
        for redo in ("0", "1"):
            os.environ["SPC_FWD_FORCE_REDO"] = redo
            Y = spc.sparse_conv_fwd(X, W, bias, "magnitude", k)
        os.environ.pop("SPC_FWD_FORCE_REDO")
        Y = Y.exact()
        dy = torch.from_numpy(grad_values(Y.nnz_bound, 7003, values="dyadic")).cuda()
        spc.sparse_conv_bwd(X, W, Y, dy)
        plan = spc.BwdPlan(X, W, Y)
        ar = spc.dp.GradAllReduce(w.nnz, co, "cuda")
        plan.f64(X, W, Y, dy, torch.empty(max(X.nnz_bound, 1), device="cuda"), ar.dw64, ar.db64)
        ar(torch.empty(w.nnz, device="cuda"), torch.empty(co, device="cuda"))
        r, src = spc.sparse_relu(Y)
        spc.sparse_scatter_grad(src, torch.ones(max(r.nnz_bound, 1), device="cuda"), r.nnz_bound, Y.nnz_bound,
                                r.nnz_dev)
        spc.sparse_scatter_grad(src, torch.ones(max(r.nnz_bound, 1), device="cuda"), r.nnz_bound, Y.nnz_bound,
                                r.nnz_dev, sorted=True)
        spc.sparse_maxpool(Y, (2,) * len(dims))
        spc.attention_topk(Y, "raw", max(1, k // 3))
    # top-k with the 13-bit first digit (segments of >= 32 Ki entries)
    x = uniform_map(1, 2, (64, 64, 64), 0.2, 7010, values="dyadic")
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
    spc.attention_topk(X, "magnitude", 20000)
    spc.attention_topk(X, "raw", 20000)
    # key codec
    co = torch.tensor([[1, 0, 2, 3], [0, 2, 3, 1], [1, 2, 0, 0]], dtype=torch.int64).cuda()
    kk = spc.encode_keys(co, 2, 3, (4, 4))
    spc.decode_keys(kk, 2, 3, (4, 4))
    # spatial sharding (f4): halo assembly, owned-plane extraction, distributed select, dx routing
    from paper_1801_10585_b200.spatial import LoopbackComm, SpatialConv, extract_planes
    x = uniform_map(2, 3, (12, 10, 14), 0.08, 7020, values="dyadic")
    w = sparse_filter(3, 4, (3, 3, 3), 0.5, 7021, values="dyadic")
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
    W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
    layer = SpatialConv(LoopbackComm(3), 12)
    xs = [extract_planes(X, a, e)[0].exact() for a, e in layer.ranges()]
    ys = [y.exact() for y in layer.forward(xs, W, None, "magnitude", 200)]
    layer.backward(xs, W, ys, [torch.ones(max(y.nnz_bound, 1), device="cuda")[:y.nnz_bound] for y in ys])
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()

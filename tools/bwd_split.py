import sys, os, json, torch
sys.path.insert(0, os.getcwd())
import paper_1801_10585_b200 as spc
from synth import uniform_map, sparse_filter, bias_vector
for d in (0.05, 0.2, 0.5):
    x = uniform_map(8, 32, (64, 64, 64), d, 123, sites="indep")
    w = sparse_filter(32, 32, (3, 3, 3), 1.0, 5)
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
    W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
    k = int(d * 64 ** 3)
    Y = spc.sparse_conv_fwd(X, W, None, "magnitude", k, variant="gemm").exact()
    dy = torch.randn(Y.nnz_bound, device="cuda")
    res = {"density": d}
    for name, fn in [("both", lambda: spc.sparse_conv_bwd(X, W, Y, dy)),
                     ("dx", lambda: spc.sparse_conv_bwd(X, W, Y, dy, need_dw=False, need_dbias=False)),
                     ("dw", lambda: spc.sparse_conv_bwd(X, W, Y, dy, need_dx=False))]:
        for _ in range(2): fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5): fn()
        b.record(); b.synchronize()
        res[name] = round(a.elapsed_time(b) / 5, 3)
    print(json.dumps(res))

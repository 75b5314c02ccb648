"""Time one C5 layer (64^3, batch 8, 32 -> 32, 3x3x3, exact conv) forward with a given variant and
print the per-phase kernel times: python tools/c5time.py DENSITY VARIANT [ITERS]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1801_10585_b200 as spc  # noqa: E402
from synth import uniform_map, sparse_filter, bias_vector  # noqa: E402

d = float(sys.argv[1])
var = sys.argv[2]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
x = uniform_map(8, 32, (64, 64, 64), d, 123, sites="indep")
w = sparse_filter(32, 32, (3, 3, 3), 1.0, 5)
X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
b = torch.from_numpy(bias_vector(32, 5)).cuda()
p = spc.FwdPlan(X, W, "none", 0, var)
for _ in range(3):
    p(X, W, b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    p(X, W, b)
e1.record()
e1.synchronize()
spc.profile_reset()
spc.profile_enable(True)
p(X, W, b)
torch.cuda.synchronize()
spc.profile_enable(False)
ph = {k: round(v[0], 4) for k, v in spc.profile_read().items()}
print(json.dumps({"density": d, "variant": p.resolved, "ms": round(e0.elapsed_time(e1) / iters, 4), "phases": ph,
                  "ksplit_env": os.environ.get("SPC_GEMM_KSPLIT", "")}))

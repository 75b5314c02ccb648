import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_1801_10585_b200 as spc
from synth import uniform_map, sparse_filter, bias_vector, SEED_BASE
d = float(sys.argv[1]); var = sys.argv[2]
x = uniform_map(8, 32, (64,64,64), d, 123, sites="indep")
w = sparse_filter(32, 32, (3,3,3), 1.0, 5)
X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
b = torch.from_numpy(bias_vector(32, 5)).cuda()
p = spc.FwdPlan(X, W, "none", 0, var)
for _ in range(3): p(X, W, b)
torch.cuda.synchronize()

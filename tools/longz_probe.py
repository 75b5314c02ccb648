"""Probe: forward / backward support and parity on long rows (1D signals, long last dimension)."""
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
import oracle as ora  # noqa: E402
import paper_1801_10585_b200 as spc  # noqa: E402
from synth import uniform_map, sparse_filter, grad_values  # noqa: E402
import torch  # noqa: E402

for dims, ci, co in [((5000,), 2, 3), ((8000,), 2, 3), ((3, 9000), 2, 3), ((40000,), 2, 3), ((40000,), 40, 3)]:
    x = uniform_map(2, ci, dims, 0.01, 9, values="dyadic")
    w = sparse_filter(ci, co, (3,) * len(dims), 0.6, 9, values="dyadic")
    X = spc.SparseMap.from_arrays(x.keys, x.values, x.batch, x.channels, x.dims)
    W = spc.SparseFilter.from_arrays(w.keys, w.values, w.c_in, w.c_out, w.ksize)
    try:
        Y = spc.sparse_conv_fwd(X, W, None, "none", 0, variant="auto")
        yk = Y.trimmed()[0].cpu().numpy().view(np.uint64)
        dy = grad_values(yk.shape[0], 10, values="dyadic")
        dx, dw, db = spc.sparse_conv_bwd(X, W, Y.exact(), torch.from_numpy(dy).cuda())
        odx, odw, _, _, _ = ora.conv_bwd(x, w, yk, dy, with_abs=True)
        print(dims, ci, "bwd", "ok" if np.array_equal(dx.cpu().numpy(), odx) else "MISMATCH")
    except Exception as e:
        print(dims, ci, "error", str(e)[:90])

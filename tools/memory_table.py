"""Table 1 / Fig. 7 next to this implementation's footprint.

For the paper's setting (3D r^3, minibatch 32, one input channel, 8 output channels, 3x3x3
filter, rho = rho_up = 1/r) it prints, in GB: the paper's formula (spc_memory_estimate: dense,
sparse 32/64, temp) and what libspconv needs for the same forward layer -- the output arrays
(capacity x 12 B) plus the workspace of sparse_conv_fwd (all samples' buffers at once) and of
sparse_conv_fwd_pass with samples_per_pass = 1. Host-side queries only (no GPU needed).

  python tools/memory_table.py [--res 32 64 128 256 512]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1801_10585_b200 as spc  # noqa: E402
from paper_1801_10585_b200._lib import FilterT, MapT  # noqa: E402


def structs(r, batch, c_in, c_out, rho):
    m = MapT()
    m.ndim, m.batch, m.channels = 3, batch, c_in
    for i in range(3):
        m.dims[i] = r
    m.nnz, m.keys, m.values = int(rho * r ** 3) * batch * c_in, 64, 64   # dummy pointers, never read
    f = FilterT()
    f.ndim, f.c_in, f.c_out = 3, c_in, c_out
    for i in range(3):
        f.ksize[i] = 3
    f.nnz, f.keys, f.values = 27 * c_in * c_out, 64, 64
    return m, f


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--res", type=int, nargs="*", default=[32, 64, 128, 256, 512])
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--c-out", type=int, default=8)
    args = ap.parse_args()
    lib = spc.load()
    rows = []
    for r in args.res:
        rho = 1.0 / r
        k = int(rho * r ** 3)
        est64 = spc.memory_estimate(3, r, args.batch, args.c_out, rho, 64)
        try:
            s32 = spc.memory_estimate(3, r, args.batch, args.c_out, rho, 32)["sparse"]
        except RuntimeError:
            s32 = None
        m, f = structs(r, args.batch, 1, args.c_out, rho)
        cap, ws_all, ws_one = C.c_int64(), C.c_size_t(), C.c_size_t()
        assert lib.spc_conv_fwd_query_pass(C.byref(m), C.byref(f), 1, k, 0, C.byref(cap), C.byref(ws_all)) == 0
        assert lib.spc_conv_fwd_query_pass(C.byref(m), C.byref(f), 1, k, 1, C.byref(cap), C.byref(ws_one)) == 0
        out = cap.value * 12
        g = 1e9
        rows.append({"r": r, "paper_dense_gb": est64["dense"] / g, "paper_sparse32_gb": None if s32 is None else s32 / g,
                     "paper_sparse64_gb": est64["sparse"] / g, "paper_temp_gb": est64["temp"] / g,
                     "ours_output_gb": out / g, "ours_ws_all_samples_gb": ws_all.value / g,
                     "ours_ws_one_sample_gb": ws_one.value / g})
    hdr = ("r", "dense", "sparse32", "sparse64", "temp", "| ours: out", "ws(all b)", "ws(1 b/pass)")
    print("%5s %9s %9s %9s %9s %11s %10s %12s" % hdr)
    for x in rows:
        print("%5d %9.4g %9s %9.4g %9.4g %11.4g %10.4g %12.4g" % (
            x["r"], x["paper_dense_gb"], "-" if x["paper_sparse32_gb"] is None else "%.4g" % x["paper_sparse32_gb"],
            x["paper_sparse64_gb"], x["paper_temp_gb"], x["ours_output_gb"], x["ours_ws_all_samples_gb"],
            x["ours_ws_one_sample_gb"]))
    print(json.dumps(rows))


if __name__ == "__main__":
    main()

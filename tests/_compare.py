"""Comparison helpers for the GPU parity tests (tolerance rule of DESIGN.md "Tolerances")."""
from __future__ import annotations

import numpy as np

REL = 1e-5      # north star: 1e-5 relative (fp32 accumulation-order differences)
ABS_SCALE = 1e-6  # times the oracle's sum of |terms| of the element (cancellation floor)


def assert_values_close(gpu, ora, abs_sum, what="values"):
    gpu = np.asarray(gpu, np.float64)
    ora = np.asarray(ora, np.float64)
    err = np.abs(gpu - ora)
    bound = REL * np.abs(ora) + ABS_SCALE * np.asarray(abs_sum, np.float64)
    bad = np.nonzero(err > bound)[0]
    assert bad.size == 0, (f"{what}: {bad.size}/{gpu.size} outside tolerance; first {bad[:5]}: gpu {gpu[bad[:5]]} "
                           f"ora {ora[bad[:5]]} bound {bound[bad[:5]]}")


def score(v, attn):
    v = np.asarray(v, np.float64)
    return np.abs(v) if attn == "magnitude" else v


def assert_topk_sets_match(gk, gv, ok, ov, all_keys, all_vals, all_abs, V, k, attn):
    """Continuous values: kept sets per segment have equal sizes and any key in the symmetric
    difference has a score within the value tolerance of the oracle's k-th score."""
    gk = np.asarray(gk, np.uint64)
    ok = np.asarray(ok, np.uint64)
    assert gk.shape == ok.shape, (gk.shape, ok.shape)
    if np.array_equal(gk, ok):
        return 0
    seg_all = (all_keys // np.uint64(V)).astype(np.int64)
    sc = score(all_vals, attn)
    lookup = {int(kk): i for i, kk in enumerate(all_keys.tolist())}
    diff = set(gk.tolist()) ^ set(ok.tolist())
    for kk in diff:
        i = lookup[int(kk)]
        s = seg_all[i]
        m = seg_all == s
        ss = np.sort(sc[m])[::-1]
        T = ss[min(k, ss.size) - 1]
        tol = 2 * (REL * abs(all_vals[i]) + ABS_SCALE * all_abs[i]) + 1e-12
        assert abs(sc[i] - T) <= tol, f"key {kk} score {sc[i]} not within {tol} of threshold {T}"
    return len(diff)

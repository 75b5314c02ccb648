"""Per-sample oracle runs in worker processes (test infrastructure). A full-size batch is too
slow for one single-threaded oracle call; samples are independent in Alg. 1 and dx, and dw is a
sum over samples (Alg. 2), so each worker runs the unmodified oracle on one sample and the
parent adds the fp64 partials in sample order before rounding once."""
from __future__ import annotations

import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np


def _one(args):
    import oracle as ora
    from synth import grad_values, select_samples

    x, w, bias, attn, k, b, dy_seed = args
    xs = select_samples(x, [b])
    yk, yv, ya, macs = ora.conv_fwd(xs, w, bias, attn=attn, k=k, with_abs=True)
    dy = grad_values(yk.shape[0], dy_seed + b)
    dx, dw64, db64, dxa, dwa = ora.conv_bwd64(xs, w, yk, dy, with_abs=True)
    return b, yk, yv, ya, dy, dx, dxa, dw64, db64, dwa


def per_sample_oracle(x, w, bias, attn, k, dy_seed, samples=None, workers=None):
    """Oracle forward (attention) and backward of each sample with dy = grad_values(n_b, dy_seed + b)
    on the sample's own kept outputs. Returns the batch-level results in key order."""
    samples = list(range(x.batch)) if samples is None else list(samples)
    workers = workers or min(len(samples), max(1, (os.cpu_count() or 2) - 1))
    import multiprocessing as mp

    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("spawn")) as ex:
        res = sorted(ex.map(_one, [(x, w, bias, attn, k, b, dy_seed) for b in samples]), key=lambda r: r[0])
    V = x.volume
    span = np.uint64(w.c_out * V)
    yk = np.concatenate([r[1] + np.uint64(i) * span for i, r in enumerate(res)])
    dw64 = np.zeros(w.nnz, np.float64)
    db64 = np.zeros(w.c_out, np.float64)
    dwa = np.zeros(w.nnz, np.float64)
    for r in res:   # fp64 partials added in sample order, rounded once by the caller
        dw64 += r[7]
        db64 += r[8]
        dwa += r[9]
    return {
        "yk": yk, "yv": np.concatenate([r[2] for r in res]), "ya": np.concatenate([r[3] for r in res]),
        "dy": np.concatenate([r[4] for r in res]), "dx": np.concatenate([r[5] for r in res]),
        "dxa": np.concatenate([r[6] for r in res]), "dw64": dw64, "db64": db64, "dwa": dwa, "workers": workers,
    }

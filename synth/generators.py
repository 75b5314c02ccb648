"""Seeded generators for the paper's workloads.

Layouts follow the boundary format (include/spconv.h):

* feature map key  = ((b*C + c) * V + row_major(p)),  V = prod(dims), first spatial dim most
  significant ("compressed into unique 1D keys", "sorted w.r.t. batches and
  within each batch w.r.t. channels"; reading R11 in DESIGN.md);
* filter key       = ((oc*c_in + ic) * prod(ksize) + row_major(delta)) (PAPER.md:45
  "filter weights are sorted w.r.t. the output channels and within each channel w.r.t. the
  input channels").

Every sample b draws from its own stream SeedSequence([seed, b]) so that a data-parallel rank
can generate only its shard and obtain exactly the rows of the full batch.

Value modes:
* "continuous": U[-1, 1] without 0;
* "dyadic": j/64 with j in [-64, 64] \\ {0}; "dyadic4": j/4 with j in [-4, 4] \\ {0} (coarse grid
  for deeper layers of a chain, so that exactness survives several layers). Products of two such values are multiples of
  2^-12; sums of fewer than 2^12 such products are exact in fp32 in any order, which makes the
  GPU and the oracle agree bit for bit.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

SEED_BASE = 180110585


@dataclass
class COO:
    """Coordinate-sorted sparse feature map."""

    batch: int
    channels: int
    dims: tuple
    keys: np.ndarray  # uint64 [nnz], strictly increasing
    values: np.ndarray  # float32 [nnz]

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def volume(self) -> int:
        return int(np.prod(self.dims))

    @property
    def nnz(self) -> int:
        return int(self.keys.shape[0])


@dataclass
class Filter:
    """Sparse filter bank, keys sorted by (oc, ic, delta)."""

    c_in: int
    c_out: int
    ksize: tuple
    keys: np.ndarray  # uint64 [nnz]
    values: np.ndarray  # float32 [nnz]

    @property
    def ndim(self) -> int:
        return len(self.ksize)

    @property
    def nnz(self) -> int:
        return int(self.keys.shape[0])


def _rng(seed: int, *path: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed) & 0xFFFFFFFF, *[int(p) for p in path]]))


def _draw_values(rng: np.random.Generator, n: int, mode: str) -> np.ndarray:
    if mode == "continuous":
        v = rng.uniform(-1.0, 1.0, size=n).astype(np.float32)
        v[v == 0] = np.float32(0.5)
        return v
    if mode == "dyadic":
        j = rng.integers(1, 65, size=n) * rng.choice(np.array([-1, 1]), size=n)
        return (j.astype(np.float32) / np.float32(64.0)).astype(np.float32)
    if mode == "dyadic4":
        j = rng.integers(1, 5, size=n) * rng.choice(np.array([-1, 1]), size=n)
        return (j.astype(np.float32) / np.float32(4.0)).astype(np.float32)
    if mode == "signed_zero":   # max-pool tie cases: +0 / -0 / negatives / positives (R8)
        pool = np.array([-1.0, -0.5, -0.0, 0.0, 0.5], np.float32)
        return pool[rng.integers(0, 5, size=n)].astype(np.float32)
    if mode == "positive":
        return rng.uniform(0.05, 1.0, size=n).astype(np.float32)
    raise ValueError(f"unknown value mode {mode!r}")


def _assemble(batch, channels, dims, per_sample) -> COO:
    """per_sample[b] = list over c of sorted int64 positions and float32 values."""
    V = int(np.prod(dims))
    keys, vals = [], []
    for b, chans in enumerate(per_sample):
        for c, (pos, v) in enumerate(chans):
            keys.append((np.uint64((b * channels + c) * V) + pos.astype(np.uint64)))
            vals.append(v)
    if keys:
        k = np.concatenate(keys).astype(np.uint64)
        v = np.concatenate(vals).astype(np.float32)
    else:
        k = np.zeros(0, np.uint64)
        v = np.zeros(0, np.float32)
    return COO(batch, channels, tuple(int(d) for d in dims), k, v)


def uniform_map(batch: int, channels: int, dims: Sequence[int], density: float, seed: int,
                values: str = "continuous", sites: str = "indep", b0: int = 0) -> COO:
    """Uniform random voxel grid ("sparse voxel grid filled with random numbers").

    `density` is per (b, c) segment: n = round(density * V) distinct positions drawn without
    replacement. sites="indep": every channel draws its own positions (paper protocol);
    sites="shared": all channels of a sample share one position set.
    """
    dims = tuple(int(d) for d in dims)
    V = int(np.prod(dims))
    n = int(round(density * V))
    n = max(0, min(V, n))
    per = []
    for bl in range(batch):
        rng = _rng(seed, b0 + bl)
        chans = []
        shared = np.sort(rng.choice(V, n, replace=False)).astype(np.int64) if sites == "shared" else None
        for _c in range(channels):
            pos = shared if shared is not None else np.sort(rng.choice(V, n, replace=False)).astype(np.int64)
            chans.append((pos, _draw_values(rng, n, values)))
        per.append(chans)
    return _assemble(batch, channels, dims, per)


def _segment_dist(P, A, B):
    """Distance from points P [...,2] to segment AB."""
    ab = B - A
    t = np.clip(((P - A) @ ab) / max(float(ab @ ab), 1e-12), 0.0, 1.0)
    proj = A + t[..., None] * ab
    return np.linalg.norm(P - proj, axis=-1)


def mnist_like(batch: int, seed: int, values: str = "mnist", b0: int = 0) -> COO:
    """Sparse MNIST-like 28x28 digits (pixels v<50 set to zero, mean density 0.23).

    2-4 strokes per image, each a polyline of 2-3 points uniform in [5, 23]^2, width
    w ~ U[1.4, 2.2], intensity round(255 * clip(1.5 - d/w, 0, 1)) with d the distance of the
    pixel centre to the polyline; images combine strokes by max; v < 50 -> 0; value v/255.
    values="dyadic" rounds v/255 to the nearest j/64 (j >= 1).
    """
    H = W = 28
    yy, xx = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(W, dtype=np.float64), indexing="ij")
    P = np.stack([yy, xx], -1)
    per = []
    for bl in range(batch):
        rng = _rng(seed, b0 + bl)
        img = np.zeros((H, W))
        for _s in range(int(rng.integers(2, 5))):
            npts = int(rng.integers(2, 4))
            pts = rng.uniform(5, 23, size=(npts, 2))
            w = rng.uniform(1.4, 2.2)
            d = np.full((H, W), np.inf)
            for i in range(npts - 1):
                d = np.minimum(d, _segment_dist(P, pts[i], pts[i + 1]))
            img = np.maximum(img, np.round(255 * np.clip(1.5 - d / w, 0, 1)))
        img[img < 50] = 0
        flat = img.reshape(-1)
        pos = np.nonzero(flat)[0].astype(np.int64)
        v = (flat[pos] / 255.0).astype(np.float32)
        if values == "dyadic":
            v = np.maximum(np.round(v * 64.0), 1.0).astype(np.float32) / np.float32(64.0)
        per.append([(pos, v.astype(np.float32))])
    return _assemble(batch, 1, (H, W), per)


def surface_occupancy(batch: int, res: int, occupancy: float, seed: int, b0: int = 0) -> COO:
    """Point-cloud-like occupancy grid ("the large majority of points lies on a
    small number of 2D surfaces"; PAPER.md:208 rho = 1/r for surfaces in a voxel grid).

    Voxelised sphere shells (radius ~ U[4, 20]) and bounded plane patches are added until the
    occupancy reaches `occupancy`; then random voxels of the last shape are dropped so that
    every sample holds exactly ceil(occupancy * res^3) occupied voxels, all with value 1.0
    (binary values: many exact ties, exercising the attention tie rule).
    """
    R = int(res)
    V = R ** 3
    target = int(np.ceil(occupancy * V))
    g = np.arange(R, dtype=np.float64)
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    per = []
    for bl in range(batch):
        rng = _rng(seed, b0 + bl)
        occ = np.zeros(V, dtype=bool)
        while True:
            if rng.random() < 0.6:
                r = rng.uniform(4, min(20, R / 2 - 1))
                c = rng.uniform(r, R - 1 - r, size=3)
                d = np.sqrt((X - c[0]) ** 2 + (Y - c[1]) ** 2 + (Z - c[2]) ** 2)
                shape = np.abs(d - r) < 0.5
            else:
                n = rng.normal(size=3)
                n /= np.linalg.norm(n)
                c = rng.uniform(0, R - 1, size=3)
                pr = rng.uniform(5, 15)
                dist = (X - c[0]) * n[0] + (Y - c[1]) * n[1] + (Z - c[2]) * n[2]
                rad = np.sqrt((X - c[0]) ** 2 + (Y - c[1]) ** 2 + (Z - c[2]) ** 2)
                shape = (np.abs(dist) < 0.5) & (rad < pr)
            new = shape.reshape(-1) & ~occ
            cnt = int(occ.sum())
            nn = int(new.sum())
            if cnt + nn >= target:
                idx = np.nonzero(new)[0]
                keep = rng.choice(idx, target - cnt, replace=False)
                occ[keep] = True
                break
            occ |= new
        pos = np.nonzero(occ)[0].astype(np.int64)
        per.append([(pos, np.ones(pos.shape[0], np.float32))])
    return _assemble(batch, 1, (R, R, R), per)


def sparse_filter(c_in: int, c_out: int, ksize: Sequence[int], density: float, seed: int,
                  values: str = "continuous", scale: float = 1.0) -> Filter:
    """Sparse filter bank with density rho_f.

    Draws a dense bank and keeps the round(density * total) largest |w| (ties by position), which
    emulates the output of the paper's magnitude pruning without training.
    `scale` multiplies the values (a power of two keeps dyadic values dyadic).
    """
    ksize = tuple(int(k) for k in ksize)
    K = int(np.prod(ksize))
    total = c_in * c_out * K
    rng = _rng(seed, 0xF11)
    w = _draw_values(rng, total, values) * np.float32(scale)
    nkeep = max(1, min(total, int(round(density * total))))
    order = np.argsort(-np.abs(w.astype(np.float64)), kind="stable")[:nkeep]
    idx = np.sort(order).astype(np.uint64)
    return Filter(int(c_in), int(c_out), ksize, idx, w[idx.astype(np.int64)].astype(np.float32))


def bias_vector(c_out: int, seed: int, values: str = "continuous") -> np.ndarray:
    """Per-output-channel bias (Alg. 1 "add bias to non-zero entries")."""
    rng = _rng(seed, 0xB1A5)
    if values == "dyadic":
        return (rng.integers(-409, 410, size=c_out).astype(np.float32) / np.float32(4096.0)).astype(np.float32)
    return rng.uniform(-0.1, 0.1, size=c_out).astype(np.float32)


def grad_values(n: int, seed: int, values: str = "continuous") -> np.ndarray:
    """Synthetic upstream gradient dL/dy on the kept output entries."""
    rng = _rng(seed, 0x6AD)
    return _draw_values(rng, n, values)


def select_samples(x: COO, samples: Sequence[int]) -> COO:
    """Sub-batch made of the given samples (re-indexed 0..len-1); used to run the oracle on a
    sample of a full-size batch. Pure re-indexing of keys (no arithmetic of the method)."""
    V = x.volume
    C = x.channels
    span = np.uint64(C * V)
    keys, vals = [], []
    for nb, b in enumerate(samples):
        lo = np.searchsorted(x.keys, np.uint64(b) * span)
        hi = np.searchsorted(x.keys, np.uint64(b + 1) * span)
        keys.append(x.keys[lo:hi] - np.uint64(b) * span + np.uint64(nb) * span)
        vals.append(x.values[lo:hi])
    return COO(len(samples), C, x.dims, np.concatenate(keys).astype(np.uint64),
               np.concatenate(vals).astype(np.float32))

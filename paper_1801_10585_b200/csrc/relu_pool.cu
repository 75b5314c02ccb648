// Sparse ReLU and sparse max-pooling (§3.3) as compacting kernels.
#include "spc_internal.cuh"
#include "block_scan.cuh"

#include <algorithm>

namespace spc {

// ------------------------------------------------------------------------------- ReLU
// Keep v > 0 (reading R9); order preserved; ordered stream compaction in two passes over
// 4096-entry chunks (count, device scan, write).
constexpr int kReluThreads = 256;
constexpr int kReluItems = 16;
constexpr int kReluChunk = kReluThreads * kReluItems;

__global__ void __launch_bounds__(kReluThreads) relu_count_kernel(const float* __restrict__ vals, const int64_t* nnz_dev,
                                                                  int64_t nbound, uint32_t* __restrict__ cnt) {
    const int64_t n = load_n(nnz_dev, nbound);
    const int64_t base = (int64_t)blockIdx.x * kReluChunk;
    uint32_t c = 0;
#pragma unroll
    for (int u = 0; u < kReluItems; ++u) {
        const int64_t i = base + (int64_t)u * kReluThreads + threadIdx.x;
        if (i < n) c += vals[i] > 0.0f;
    }
    __shared__ uint32_t sm[33];
    const uint32_t tot = block_sum(c, sm);
    if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

// Write pass: warp w of a chunk owns its 512 consecutive entries (16 groups of 32, coalesced);
// one ballot per group gives each kept entry its slot, warp totals are scanned across the block,
// and keys / values / source indices are stored with consecutive addresses per group.
__global__ void __launch_bounds__(kReluThreads) relu_write_kernel(Keys keys,
                                                                  const float* __restrict__ vals, const int64_t* nnz_dev,
                                                                  int64_t nbound, const uint64_t* __restrict__ off,
                                                                  KeysOut ok, float* __restrict__ ov,
                                                                  int64_t* __restrict__ osrc) {
    const int64_t n = load_n(nnz_dev, nbound);
    const int64_t base = (int64_t)blockIdx.x * kReluChunk;
    if (base >= n) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t w0 = base + (int64_t)warp * (32 * kReluItems);
    const uint64_t pos0 = off[blockIdx.x];   // in flight with the value loads
    // values and keys in one round trip (the keys' sectors are fetched anyway at these kept
    // fractions), in flight during the block-wide scan
    float v[kReluItems];
    uint64_t k[kReluItems];
#pragma unroll
    for (int u = 0; u < kReluItems; ++u) {
        const int64_t i = w0 + 32 * u + lane;
        v[u] = i < n ? vals[i] : 0.0f;
        k[u] = i < n ? keys[i] : 0ull;
    }
    unsigned m[kReluItems];
    uint32_t c = 0;
#pragma unroll
    for (int u = 0; u < kReluItems; ++u) {
        m[u] = __ballot_sync(kFull, v[u] > 0.0f);
        c += (uint32_t)__popc(m[u]);
    }
    __shared__ uint32_t wc[kReluThreads / 32];
    if (lane == 0) wc[warp] = c;
    __syncthreads();
    uint64_t pos = pos0;
    for (int q = 0; q < warp; ++q) pos += wc[q];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int u = 0; u < kReluItems; ++u) {
        if (v[u] > 0.0f) {
            const int64_t i = w0 + 32 * u + lane;
            const uint64_t o = pos + (uint32_t)__popc(m[u] & lt);
            ok.put(o, k[u]);
            ov[o] = v[u];
            if (osrc) osrc[o] = i;
        }
        pos += (uint32_t)__popc(m[u]);
    }
}

cudaError_t launch_relu(Keys keys, const float* vals, const int64_t* nnz_dev, int64_t nbound,
                        uint32_t* chunk_cnt, uint64_t* chunk_off, uint64_t* scan_tmp,
                        KeysOut out_keys, float* out_vals, int64_t* out_src, int64_t* out_nnz, cudaStream_t s) {
    const int64_t nch = (nbound + kReluChunk - 1) / kReluChunk;
    if (nch == 0) return cudaMemsetAsync(out_nnz, 0, sizeof(int64_t), s);
    { SPC_PHASE("relu_count", s, 1); relu_count_kernel<<<(unsigned)nch, kReluThreads, 0, s>>>(vals, nnz_dev, nbound, chunk_cnt); }
    cudaError_t e = launch_scan_u32(chunk_cnt, chunk_off, nch, out_nnz, scan_tmp, s);
    if (e != cudaSuccess) return e;
    { SPC_PHASE("relu_write", s, 1); relu_write_kernel<<<(unsigned)nch, kReluThreads, 0, s>>>(keys, vals, nnz_dev, nbound, chunk_off, out_keys,
                                                             out_vals, out_src); }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------- max-pool
// §3.3: "features are assigned to an output (hyper-) voxel, by dividing ... their index by
// strides", then the max is taken per cluster. The paper sorts by voxel (Eq. (2),
// O(n log n)); here every pooled row segment (b, c, X', Y', z-chunk) is one warp work item:
// its clusters receive the members from the sx*sy contributing input rows through native
// shared-memory integer atomics (max on an order-preserving u32 of the value, then min of
// the entry index among the maxima = smaller key wins, reading R8), and the occupied
// clusters are compacted in pooled-key order. No sort.
constexpr int kPoolThreads = 256;
constexpr int kPoolWarps = kPoolThreads / 32;
constexpr int kPoolZChunk = 512;

// Tile form (the usual case, PZ <= 4096 and a band's key span < 2^31): the inputs of the pooled
// rows py0 .. py0+nyb-1 of one pooled plane are sx contiguous key runs (one per input plane x,
// rows py0*sy .. (py0+nyb)*sy - 1), so one CTA streams them with coalesced loads into a
// shared-memory tile of nyb x PZ clusters and writes the occupied clusters in pooled-key order.
constexpr int kTileThreads = 256;
constexpr int kTileCells = 4096;

PoolPlan plan_pool(const Geo& g, int sw, int sx, int sy, int sz) {
    PoolPlan p{};
    p.sw = sw; p.sx = sx; p.sy = sy; p.sz = sz;
    p.PW = (g.W + sw - 1) / sw;
    p.PX = (g.X + sx - 1) / sx;
    p.PY = (g.Y + sy - 1) / sy;
    p.PZ = (g.Z + sz - 1) / sz;
    p.zchunk = p.PZ < kPoolZChunk ? p.PZ : kPoolZChunk;
    p.nzc = (p.PZ + p.zchunk - 1) / p.zchunk;
    p.items = g.B * g.C * (int64_t)p.PW * p.PX * p.PY * p.nzc;
    if (p.PZ <= kTileCells) {
        p.nyb = std::max(1, std::min(p.PY, kTileCells / p.PZ));
        if ((uint64_t)p.nyb * sy * (uint64_t)g.Z < (1ull << 31) && sw * sx <= 64) {   // (kMemPlanes)
            p.tiled = 1;
            p.nyt = (p.PY + p.nyb - 1) / p.nyb;
            p.mZ = ~0u / (uint32_t)g.Z;
            p.msy = ~0u / (uint32_t)sy;
            p.msz = ~0u / (uint32_t)sz;
            auto lg = [](int64_t d) { int l = 0; while ((1ll << l) < d) ++l; return (1ll << l) == d ? l : -1; };
            p.lZ = lg(g.Z);
            p.lsy = lg(sy);
            p.lsz = lg(sz);
            p.items = g.B * g.C * (int64_t)p.PW * p.PX * p.nyt;
        }
    }
    return p;
}

size_t pool_bound_words(const Geo& g, const PoolPlan& p) {
    return p.tiled ? (size_t)(g.B * g.C * (int64_t)g.W * g.X * (p.nyt + 1)) : (size_t)(g.B * g.C * g.R + 1);
}

// x / d for x < 2^31 with m = floor((2^32 - 1) / d): the multiply-high is exact or one short
__device__ __forceinline__ uint32_t udiv(uint32_t x, uint32_t d, uint32_t m) {
    uint32_t q = __umulhi(x, m);
    return (q + 1) * d <= x ? q + 1 : q;
}

// member entries of a tile: the sx key runs, four loads in flight per thread;
// f(cell, entry, value) for each (value loaded only when LOADV)
// Band bounds of the tile form: bnd[pl*(nyt+1) + j] = first entry of input plane pl = (seg, w, x)
// at or after input row j*nyb*sy (one binary search each, all in parallel) -- the tiles need only
// these, not the map's full row index.
__global__ void pool_bounds_kernel(Geo g, PoolPlan p, Keys keys, const int64_t* nnz_dev, int64_t nbound,
                                   uint32_t* __restrict__ bnd) {
    const int64_t nb = (int64_t)p.nyt + 1;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t npl = g.B * g.C * (int64_t)g.W * g.X;
    if (i >= npl * nb) return;
    const int64_t pl = i / nb;
    const int j = (int)(i - pl * nb);
    const int64_t y = min((int64_t)j * p.nyb * p.sy, (int64_t)g.Y);
    const uint64_t want = (uint64_t)(pl * g.Y + y) * (uint64_t)g.Z;
    const int64_t n = load_n(nnz_dev, nbound);
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < want) lo = mid + 1; else hi = mid;
    }
    bnd[i] = (uint32_t)lo;
}

struct PoolTileId {
    int64_t seg;
    int pw, px, py0, npy, ya, yb, yt;
};
__device__ __forceinline__ PoolTileId pool_tile_id(const Geo& g, const PoolPlan& p, int64_t tile) {
    PoolTileId t;   // (tile < 2^31: a grid index; 32-bit divisions)
    const uint32_t tl = (uint32_t)tile;
    const uint32_t r0 = tl / (uint32_t)p.nyt, yt = tl - r0 * (uint32_t)p.nyt;
    const uint32_t r1 = r0 / (uint32_t)p.PX;
    t.px = (int)(r0 - r1 * (uint32_t)p.PX);
    const uint32_t r2 = r1 / (uint32_t)p.PW;
    t.pw = (int)(r1 - r2 * (uint32_t)p.PW);
    t.seg = (int64_t)r2;
    t.yt = (int)yt;
    t.py0 = t.yt * p.nyb;
    t.npy = min(p.nyb, p.PY - t.py0);
    t.ya = t.py0 * p.sy;
    t.yb = min((t.py0 + t.npy) * p.sy, g.Y);
    return t;
}


// Member entries of a tile: the runs of the sw * sx input planes (w, x) (band bounds from
// pool_bounds_kernel) as one list. pool_tile_runs fills the shared run table (starts, prefix,
// first keys) and returns the list length; pool_round loads up to kMemU list positions per
// thread (b0 + u * blockDim.x), all loads in flight before any is used, and gives each its
// pooled cell (-1: none), entry index and value (loaded only when LOADV).
constexpr int kMemU = 8;
constexpr int kMemPlanes = 64;   // (plan_pool's tile-form limit on sw * sx)
struct PoolRuns {
    uint32_t rs[kMemPlanes], rp[kMemPlanes + 1];
    unsigned long long rk[kMemPlanes];
};

__device__ __forceinline__ uint32_t pool_tile_runs(const Geo& g, const PoolPlan& p, const uint32_t* __restrict__ bnd,
                                                   const PoolTileId& t, PoolRuns& R) {
    const int np = p.sw * p.sx;
    const int tid = threadIdx.x;
    if (tid < np) {
        const int w = t.pw * p.sw + tid / p.sx, x = t.px * p.sx + tid % p.sx;
        uint32_t e0 = 0u, e1 = 0u;
        unsigned long long kb = 0ull;
        if (w < g.W && x < g.X) {
            const int64_t pl = (t.seg * g.W + w) * g.X + x;
            e0 = bnd[pl * (p.nyt + 1) + t.yt];
            e1 = bnd[pl * (p.nyt + 1) + t.yt + 1];
            kb = (unsigned long long)(pl * (int64_t)g.Y + t.ya) * (uint32_t)g.Z;
        }
        R.rs[tid] = e0;
        R.rp[tid + 1] = e1 - e0;
        R.rk[tid] = kb;
    }
    __syncthreads();
    if (tid == 0) {
        R.rp[0] = 0u;
        for (int i = 1; i <= np; ++i) R.rp[i] += R.rp[i - 1];
    }
    __syncthreads();
    return R.rp[np];
}

template <bool LOADV>
__device__ __forceinline__ void pool_round(const Geo& g, const PoolPlan& p, Keys keys, const float* __restrict__ vals,
                                           const PoolRuns& R, uint32_t total, uint32_t b0, int (&cell)[kMemU],
                                           uint32_t (&ee)[kMemU], float (&vv)[kMemU]) {
    const uint32_t Z = (uint32_t)g.Z;
    uint64_t kk[kMemU];
    int rr[kMemU];
    int r = 0;   // (a thread's list positions increase with u: the run search continues)
#pragma unroll
    for (int u = 0; u < kMemU; ++u) {
        const uint32_t q = b0 + (uint32_t)u * blockDim.x;
        rr[u] = -1;
        kk[u] = 0ull;
        vv[u] = 0.0f;
        ee[u] = 0u;
        if (q < total) {
            while (R.rp[r + 1] <= q) ++r;
            rr[u] = r;
            ee[u] = R.rs[r] + (q - R.rp[r]);
            kk[u] = keys[ee[u]];
            if (LOADV) vv[u] = vals[ee[u]];
        }
    }
#pragma unroll
    for (int u = 0; u < kMemU; ++u) {
        cell[u] = -1;
        if (rr[u] < 0) continue;
        const uint32_t rel = (uint32_t)(kk[u] - R.rk[rr[u]]);
        const uint32_t yy = p.lZ >= 0 ? rel >> p.lZ : udiv(rel, Z, p.mZ), zz = rel - yy * Z;
        const uint32_t cy = p.lsy >= 0 ? yy >> p.lsy : udiv(yy, (uint32_t)p.sy, p.msy);
        const uint32_t cz = p.lsz >= 0 ? zz >> p.lsz : udiv(zz, (uint32_t)p.sz, p.msz);
        cell[u] = (int)cy * p.PZ + (int)cz;
    }
}

// count pass: occupied clusters of the tile (a 4096-bit occupancy mask)
__global__ void __launch_bounds__(kTileThreads)
pool_tile_count_kernel(Geo g, PoolPlan p, Keys keys, const uint32_t* __restrict__ row_ptr,
                       uint32_t* __restrict__ item_cnt) {
    __shared__ uint32_t occ[kTileCells / 32];
    __shared__ uint32_t sm[33];
    __shared__ PoolRuns R;
    const PoolTileId t = pool_tile_id(g, p, blockIdx.x);
    if (threadIdx.x < kTileCells / 32) occ[threadIdx.x] = 0u;
    const uint32_t total = pool_tile_runs(g, p, row_ptr, t, R);
    for (uint32_t b0 = threadIdx.x; b0 < total; b0 += kMemU * kTileThreads) {
        int cell[kMemU];
        uint32_t ee[kMemU];
        float vv[kMemU];
        pool_round<false>(g, p, keys, nullptr, R, total, b0, cell, ee, vv);
#pragma unroll
        for (int u = 0; u < kMemU; ++u)
            if (cell[u] >= 0) atomicOr(&occ[cell[u] >> 5], 1u << (cell[u] & 31));
    }
    __syncthreads();
    const uint32_t c = threadIdx.x < kTileCells / 32 ? (uint32_t)__popc(occ[threadIdx.x]) : 0u;
    const uint32_t tot = block_sum(c, sm);
    if (threadIdx.x == 0) item_cnt[blockIdx.x] = tot;
}

// The reduction of a tile into its clusters: the maximum's order-preserving code per cluster by
// a native 32-bit shared atomicMax, then -- after a barrier -- the smallest entry index among
// the members that reached it by atomicMin (ties to the smaller key, reading R8). (A single
// 64-bit max of (code << 32 | ~entry) compiles to a CAS loop on shared memory.) One round of up
// to kMemU * 256 members keeps them in registers across the barrier; larger tiles reload.
__device__ __forceinline__ void pool_tile_reduce(const Geo& g, const PoolPlan& p, Keys keys,
                                                 const float* __restrict__ vals, const PoolRuns& R, uint32_t total,
                                                 uint32_t* bval, uint32_t* bidx, uint32_t* occ) {
    int cell[kMemU];
    uint32_t ee[kMemU];
    float vv[kMemU];
    const bool one = total <= (uint32_t)(kMemU * kTileThreads);
    for (uint32_t b0 = threadIdx.x; b0 < total; b0 += kMemU * kTileThreads) {
        pool_round<true>(g, p, keys, vals, R, total, b0, cell, ee, vv);
#pragma unroll
        for (int u = 0; u < kMemU; ++u)
            if (cell[u] >= 0) {
                atomicMax(&bval[cell[u]], orderable(vv[u]));
                atomicOr(&occ[cell[u] >> 5], 1u << (cell[u] & 31));
            }
    }
    __syncthreads();
    if (one) {
        if (threadIdx.x < total) {
#pragma unroll
            for (int u = 0; u < kMemU; ++u)
                if (cell[u] >= 0 && bval[cell[u]] == orderable(vv[u])) atomicMin(&bidx[cell[u]], ee[u]);
        }
    } else {
        for (uint32_t b0 = threadIdx.x; b0 < total; b0 += kMemU * kTileThreads) {
            pool_round<true>(g, p, keys, vals, R, total, b0, cell, ee, vv);
#pragma unroll
            for (int u = 0; u < kMemU; ++u)
                if (cell[u] >= 0 && bval[cell[u]] == orderable(vv[u])) atomicMin(&bidx[cell[u]], ee[u]);
        }
    }
    __syncthreads();
}

// the occupied clusters of the tile in cell order from the occupancy mask (threads 0..127 own
// one mask word each: exclusive scan of the popcounts, then the word's clusters are listed);
// returns the tile's cluster count
__device__ __forceinline__ uint32_t pool_tile_list(const uint32_t* occ, uint16_t* cells, uint32_t* wsum) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t w = 0, c = 0, pre = 0;
    if (warp < 4) {
        w = occ[tid];
        c = (uint32_t)__popc(w);
        pre = warp_incl_scan(c) - c;
        if (lane == 31) wsum[warp] = pre + c;
    }
    __syncthreads();
    if (warp < 4) {
        for (int q = 0; q < warp; ++q) pre += wsum[q];
        while (w) {
            const int bit = __ffs(w) - 1;
            w &= w - 1;
            cells[pre++] = (uint16_t)(tid * 32 + bit);
        }
    }
    return wsum[0] + wsum[1] + wsum[2] + wsum[3];
}

// write of the tile's clusters at output offset o0 with coalesced stores: the maximum's value
// from its order-preserving code; +-0 (the code cannot tell them apart) from the entry itself
__device__ __forceinline__ void pool_tile_out(const PoolPlan& p, const PoolTileId& t, const float* __restrict__ vals,
                                              const uint32_t* bval, const uint32_t* bidx, const uint16_t* cells,
                                              uint32_t tot, uint64_t o0, KeysOut ok, float* __restrict__ ov,
                                              int64_t* __restrict__ oarg) {
    const uint64_t pbase = ((uint64_t)((t.seg * p.PW + t.pw) * p.PX + t.px) * p.PY + t.py0) * (uint64_t)p.PZ;
    for (uint32_t q = threadIdx.x; q < tot; q += kTileThreads) {
        const uint32_t cell = cells[q];
        const uint32_t a = bidx[cell];
        const float mv = from_orderable(bval[cell]);
        ok.put(o0 + q, pbase + cell);
        ov[o0 + q] = mv != 0.0f ? mv : vals[a];
        if (oarg) oarg[o0 + q] = a;
    }
}

__device__ __forceinline__ void pool_tile_init(uint32_t* bval, uint32_t* bidx, uint32_t* occ) {
    const int tid = threadIdx.x;
    uint4* v4 = reinterpret_cast<uint4*>(bval);
    uint4* i4 = reinterpret_cast<uint4*>(bidx);
#pragma unroll
    for (int j = 0; j < kTileCells / 4 / kTileThreads; ++j) {
        v4[tid + kTileThreads * j] = make_uint4(0u, 0u, 0u, 0u);
        i4[tid + kTileThreads * j] = make_uint4(~0u, ~0u, ~0u, ~0u);
    }
    if (tid < kTileCells / 32) occ[tid] = 0u;
}

// write pass (after the count pass and the scan of the tile counts)
__global__ void __launch_bounds__(kTileThreads)
pool_tile_write_kernel(Geo g, PoolPlan p, Keys keys, const float* __restrict__ vals,
                       const uint32_t* __restrict__ row_ptr, const uint64_t* __restrict__ item_off,
                       KeysOut ok, float* __restrict__ ov, int64_t* __restrict__ oarg) {
    __shared__ __align__(16) uint32_t bval[kTileCells];
    __shared__ __align__(16) uint32_t bidx[kTileCells];
    __shared__ uint32_t occ[kTileCells / 32];
    __shared__ uint16_t cells[kTileCells];
    __shared__ uint32_t wsum[4];
    __shared__ PoolRuns R;
    const PoolTileId t = pool_tile_id(g, p, blockIdx.x);
    pool_tile_init(bval, bidx, occ);
    const uint32_t total = pool_tile_runs(g, p, row_ptr, t, R);
    pool_tile_reduce(g, p, keys, vals, R, total, bval, bidx, occ);
    const uint32_t tot = pool_tile_list(occ, cells, wsum);
    __syncthreads();
    pool_tile_out(p, t, vals, bval, bidx, cells, tot, item_off[blockIdx.x], ok, ov, oarg);
}

template <bool WRITE>
__global__ void __launch_bounds__(kPoolThreads)
pool_kernel(Geo g, PoolPlan p, Keys keys, const float* __restrict__ vals,
            const uint32_t* __restrict__ row_ptr, uint32_t* __restrict__ item_cnt,
            const uint64_t* __restrict__ item_off, KeysOut ok, float* __restrict__ ov,
            int64_t* __restrict__ oarg) {
    __shared__ uint32_t s_best[kPoolWarps][kPoolZChunk];
    __shared__ uint32_t s_arg[kPoolWarps][kPoolZChunk];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t item = (int64_t)blockIdx.x * kPoolWarps + warp;
    if (item >= p.items) return;
    uint32_t* best = s_best[warp];
    uint32_t* arg = s_arg[warp];
    const int zc = (int)(item % p.nzc);
    int64_t r = item / p.nzc;
    const int py = (int)(r % p.PY);
    r /= p.PY;
    const int px = (int)(r % p.PX);
    r /= p.PX;
    const int pw = (int)(r % p.PW);
    const int64_t seg = r / p.PW;
    const int z0 = zc * p.zchunk;
    const int nz = min(p.zchunk, p.PZ - z0);
    for (int i = lane; i < nz; i += 32) {
        best[i] = 0u;
        arg[i] = 0xffffffffu;
    }
    __syncwarp();
    const int wa = pw * p.sw, wb = min(wa + p.sw, g.W);
    const int xa = px * p.sx, xb = min(xa + p.sx, g.X);
    const int ya = py * p.sy, yb = min(ya + p.sy, g.Y);
    // pass 1: max per cluster (or occupancy only when counting)
    for (int wx = 0; wx < (wb - wa) * (xb - xa); ++wx) {
        const int w = wa + wx / (xb - xa), x = xa + wx % (xb - xa);
        for (int y = ya; y < yb; ++y) {
            const int64_t row = ((seg * g.W + w) * g.X + x) * (int64_t)g.Y + y;
            const uint32_t e0 = row_ptr[row], e1 = row_ptr[row + 1];
            const uint64_t rowbase = (uint64_t)row * (uint64_t)g.Z;
            for (uint32_t e = e0 + lane; e < e1; e += 32) {
                const int pz = (int)(keys[e] - rowbase) / p.sz - z0;
                if (pz < 0 || pz >= nz) continue;
                if (WRITE) atomicMax(&best[pz], orderable(vals[e]));
                else best[pz] = 1u;
            }
        }
    }
    __syncwarp();
    if (!WRITE) {
        uint32_t c = 0;
        for (int i = lane; i < nz; i += 32) c += best[i] != 0u;
        c = warp_sum(c);
        if (lane == 0) item_cnt[item] = c;
        return;
    }
    // pass 2: smallest entry index among the maxima (argmax, ties -> smaller key)
    for (int wx = 0; wx < (wb - wa) * (xb - xa); ++wx) {
        const int w = wa + wx / (xb - xa), x = xa + wx % (xb - xa);
        for (int y = ya; y < yb; ++y) {
            const int64_t row = ((seg * g.W + w) * g.X + x) * (int64_t)g.Y + y;
            const uint32_t e0 = row_ptr[row], e1 = row_ptr[row + 1];
            const uint64_t rowbase = (uint64_t)row * (uint64_t)g.Z;
            for (uint32_t e = e0 + lane; e < e1; e += 32) {
                const int pz = (int)(keys[e] - rowbase) / p.sz - z0;
                if (pz < 0 || pz >= nz) continue;
                if (orderable(vals[e]) == best[pz]) atomicMin(&arg[pz], e);
            }
        }
    }
    __syncwarp();
    uint64_t pos = item_off[item];
    const uint64_t pbase = ((uint64_t)((seg * p.PW + pw) * p.PX + px) * p.PY + py) * (uint64_t)p.PZ + z0;
    for (int i0 = 0; i0 < nz; i0 += 32) {
        const int i = i0 + lane;
        const bool occ = i < nz && best[i] != 0u;
        const unsigned m = __ballot_sync(kFull, occ);
        if (occ) {
            const uint64_t o = pos + __popc(m & ((1u << lane) - 1u));
            const uint32_t a = arg[i];
            ok.put(o, pbase + i);
            ov[o] = vals[a];
            if (oarg) oarg[o] = a;
        }
        pos += __popc(m);
    }
}

cudaError_t launch_maxpool(const Geo& g, const PoolPlan& p, Keys keys, const float* vals, const int64_t* nnz_dev,
                           int64_t nbound, const uint32_t* row_ptr, uint32_t* item_cnt, uint64_t* item_off, uint64_t* scan_tmp,
                           KeysOut out_keys, float* out_vals, int64_t* out_arg, int64_t* out_nnz, cudaStream_t s) {
    if (p.items == 0) return cudaMemsetAsync(out_nnz, 0, sizeof(int64_t), s);
    if (p.tiled) {   // row_ptr holds the band bounds (pool_bounds_kernel), not a row index
        const unsigned tg = (unsigned)p.items;
        {
            const int64_t nbnd = g.B * g.C * (int64_t)g.W * g.X * (p.nyt + 1);
            SPC_PHASE("pool_bounds", s, 1);
            pool_bounds_kernel<<<(unsigned)((nbnd + 255) / 256), 256, 0, s>>>(g, p, keys, nnz_dev, nbound,
                                                                              const_cast<uint32_t*>(row_ptr));
        }
        { SPC_PHASE("pool_count", s, 1); pool_tile_count_kernel<<<tg, kTileThreads, 0, s>>>(g, p, keys, row_ptr, item_cnt); }
        cudaError_t e = launch_scan_u32(item_cnt, item_off, p.items, out_nnz, scan_tmp, s);
        if (e != cudaSuccess) return e;
        { SPC_PHASE("pool_write", s, 1); pool_tile_write_kernel<<<tg, kTileThreads, 0, s>>>(g, p, keys, vals, row_ptr, item_off, out_keys, out_vals, out_arg); }
        return cudaGetLastError();
    }
    const unsigned grid = (unsigned)((p.items + kPoolWarps - 1) / kPoolWarps);
    { SPC_PHASE("pool_count", s, 1); pool_kernel<false><<<grid, kPoolThreads, 0, s>>>(g, p, keys, vals, row_ptr, item_cnt, nullptr, nullptr, nullptr,
                                                     nullptr); }
    cudaError_t e = launch_scan_u32(item_cnt, item_off, p.items, out_nnz, scan_tmp, s);
    if (e != cudaSuccess) return e;
    { SPC_PHASE("pool_write", s, 1); pool_kernel<true><<<grid, kPoolThreads, 0, s>>>(g, p, keys, vals, row_ptr, item_cnt, item_off, out_keys, out_vals,
                                                    out_arg); }
    return cudaGetLastError();
}

}  // namespace spc

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
__global__ void __launch_bounds__(kReluThreads) relu_write_kernel(const uint64_t* __restrict__ keys,
                                                                  const float* __restrict__ vals, const int64_t* nnz_dev,
                                                                  int64_t nbound, const uint64_t* __restrict__ off,
                                                                  uint64_t* __restrict__ ok, float* __restrict__ ov,
                                                                  int64_t* __restrict__ osrc) {
    const int64_t n = load_n(nnz_dev, nbound);
    const int64_t base = (int64_t)blockIdx.x * kReluChunk;
    if (base >= n) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t w0 = base + (int64_t)warp * (32 * kReluItems);
    const uint64_t pos0 = off[blockIdx.x];   // in flight with the value loads
    float v[kReluItems];
#pragma unroll
    for (int u = 0; u < kReluItems; ++u) {
        const int64_t i = w0 + 32 * u + lane;
        v[u] = i < n ? vals[i] : 0.0f;
    }
    // keys of the kept entries are loaded before the block-wide scan so that their latency
    // overlaps it
    uint64_t k[kReluItems];
    unsigned m[kReluItems];
    uint32_t c = 0;
#pragma unroll
    for (int u = 0; u < kReluItems; ++u) {
        const int64_t i = w0 + 32 * u + lane;
        k[u] = v[u] > 0.0f ? keys[i] : 0ull;
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
            ok[o] = k[u];
            ov[o] = v[u];
            if (osrc) osrc[o] = i;
        }
        pos += (uint32_t)__popc(m[u]);
    }
}

cudaError_t launch_relu(const uint64_t* keys, const float* vals, const int64_t* nnz_dev, int64_t nbound,
                        uint32_t* chunk_cnt, uint64_t* chunk_off, uint64_t* scan_tmp,
                        uint64_t* out_keys, float* out_vals, int64_t* out_src, int64_t* out_nnz, cudaStream_t s) {
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

// Tile form (the usual case, PZ <= 4096 and a band's key span < 2^32): the inputs of the pooled
// rows py0 .. py0+nyb-1 of one pooled plane are sx contiguous key runs (one per input plane x,
// rows py0*sy .. (py0+nyb)*sy - 1), so one CTA streams them with coalesced loads into a
// shared-memory tile of nyb x PZ clusters and writes the occupied clusters in pooled-key order.
constexpr int kTileThreads = 256;
constexpr int kTileCells = 4096;
constexpr int kTileJ = kTileCells / kTileThreads;   // 16 clusters per thread, cell = tid + 256 j

PoolPlan plan_pool(const Geo& g, int sx, int sy, int sz) {
    PoolPlan p{};
    p.sx = sx; p.sy = sy; p.sz = sz;
    p.PX = (g.X + sx - 1) / sx;
    p.PY = (g.Y + sy - 1) / sy;
    p.PZ = (g.Z + sz - 1) / sz;
    p.zchunk = p.PZ < kPoolZChunk ? p.PZ : kPoolZChunk;
    p.nzc = (p.PZ + p.zchunk - 1) / p.zchunk;
    p.items = g.B * g.C * (int64_t)p.PX * p.PY * p.nzc;
    if (p.PZ <= kTileCells) {
        p.nyb = std::max(1, std::min(p.PY, kTileCells / p.PZ));
        if ((uint64_t)p.nyb * sy * (uint64_t)g.Z < (1ull << 31)) {
            p.tiled = 1;
            p.nyt = (p.PY + p.nyb - 1) / p.nyb;
            p.mZ = ~0u / (uint32_t)g.Z;
            p.msy = ~0u / (uint32_t)sy;
            p.msz = ~0u / (uint32_t)sz;
            p.items = g.B * g.C * (int64_t)p.PX * p.nyt;
        }
    }
    return p;
}

// x / d for x < 2^31 with m = floor((2^32 - 1) / d): the multiply-high is exact or one short
__device__ __forceinline__ uint32_t udiv(uint32_t x, uint32_t d, uint32_t m) {
    uint32_t q = __umulhi(x, m);
    return (q + 1) * d <= x ? q + 1 : q;
}

template <bool WRITE>
__global__ void __launch_bounds__(kTileThreads)
pool_tile_kernel(Geo g, PoolPlan p, const uint64_t* __restrict__ keys, const float* __restrict__ vals,
                 const uint32_t* __restrict__ row_ptr, uint32_t* __restrict__ item_cnt,
                 const uint64_t* __restrict__ item_off, uint64_t* __restrict__ ok, float* __restrict__ ov,
                 int64_t* __restrict__ oarg) {
    __shared__ uint32_t best[kTileCells];
    __shared__ uint32_t arg[kTileCells];
    __shared__ uint32_t wcnt[kTileJ * 8 + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tile = blockIdx.x;
    const int yt = (int)(tile % p.nyt);
    const int64_t r = tile / p.nyt;
    const int px = (int)(r % p.PX);
    const int64_t seg = r / p.PX;
    const int py0 = yt * p.nyb, npy = min(p.nyb, p.PY - py0);
    const int ncell = npy * p.PZ;
#pragma unroll
    for (int j = 0; j < kTileJ; ++j) {
        best[tid + kTileThreads * j] = 0u;
        if (WRITE) arg[tid + kTileThreads * j] = 0xffffffffu;
    }
    __syncthreads();
    const int ya = py0 * p.sy, yb = min((py0 + npy) * p.sy, g.Y);
    const uint32_t Z = (uint32_t)g.Z;
    // f(cell, entry, value) over the member entries: the sx key runs, four loads in flight per thread
    auto for_members = [&](auto f) {
        for (int dx = 0; dx < p.sx; ++dx) {
            const int x = px * p.sx + dx;
            if (x >= g.X) break;
            const int64_t row0 = (seg * g.X + x) * (int64_t)g.Y + ya;
            const uint32_t e0 = row_ptr[row0], e1 = row_ptr[row0 + (yb - ya)];
            const uint64_t kb = (uint64_t)row0 * Z;
            for (uint32_t e = e0 + tid; e < e1; e += 4 * kTileThreads) {
                uint64_t kk[4];
                float vv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t ee = e + (uint32_t)u * kTileThreads;
                    kk[u] = ee < e1 ? keys[ee] : kb;
                    vv[u] = (WRITE && ee < e1) ? vals[ee] : 0.0f;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t ee = e + (uint32_t)u * kTileThreads;
                    if (ee < e1) {
                        const uint32_t rel = (uint32_t)(kk[u] - kb);
                        const uint32_t yy = udiv(rel, Z, p.mZ), zz = rel - yy * Z;
                        f((int)udiv(yy, (uint32_t)p.sy, p.msy) * p.PZ + (int)udiv(zz, (uint32_t)p.sz, p.msz), ee, vv[u]);
                    }
                }
            }
        }
    };
    // pass 1: max per cluster on an order-preserving u32 (occupancy only when counting)
    for_members([&](int cell, uint32_t, float v) {
        if (WRITE) atomicMax(&best[cell], orderable(v));
        else best[cell] = 1u;
    });
    __syncthreads();
    if (!WRITE) {
        uint32_t c = 0;
#pragma unroll
        for (int j = 0; j < kTileJ; ++j) c += best[tid + kTileThreads * j] != 0u;
        __shared__ uint32_t sm[33];
        c = block_sum(c, sm);
        if (tid == 0) item_cnt[tile] = c;
        return;
    }
    // pass 2 (the runs are L1/L2-resident now): smallest entry index among the maxima
    for_members([&](int cell, uint32_t e, float v) {
        if (orderable(v) == best[cell]) atomicMin(&arg[cell], e);
    });
    __syncthreads();
    // ordered compaction of the occupied clusters (cell order = (j, warp, lane)): one ballot per
    // j, a scan of the 16 x 8 (j, warp) counts, then the (cell, arg) pairs are staged in place
    // and written with coalesced stores
    unsigned m[kTileJ];
    uint32_t av[kTileJ];
#pragma unroll
    for (int j = 0; j < kTileJ; ++j) {
        const int cell = tid + kTileThreads * j;
        const bool occ = cell < ncell && best[cell] != 0u;
        m[j] = __ballot_sync(kFull, occ);
        av[j] = arg[cell];
        if (lane == 0) wcnt[j * 8 + warp] = (uint32_t)__popc(m[j]);
    }
    __syncthreads();
    if (warp == 0) {   // exclusive scan of the 128 counts, 4 per lane
        uint32_t c[4], t = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) { c[q] = wcnt[4 * lane + q]; t += c[q]; }
        const uint32_t inc = warp_incl_scan(t);
        uint32_t run = inc - t;
#pragma unroll
        for (int q = 0; q < 4; ++q) { wcnt[4 * lane + q] = run; run += c[q]; }
        if (lane == 31) wcnt[kTileJ * 8] = inc;
    }
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < kTileJ; ++j) {
        if ((m[j] >> lane) & 1u) {
            const uint32_t q = wcnt[j * 8 + warp] + (uint32_t)__popc(m[j] & lt);
            best[q] = (uint32_t)(tid + kTileThreads * j);
            arg[q] = av[j];
        }
    }
    const uint32_t tot = wcnt[kTileJ * 8];
    __syncthreads();
    const uint64_t o0 = item_off[tile];
    const uint64_t pbase = ((uint64_t)(seg * p.PX + px) * p.PY + py0) * (uint64_t)p.PZ;
    for (uint32_t q = tid; q < tot; q += kTileThreads) {
        const uint32_t a = arg[q];
        ok[o0 + q] = pbase + best[q];
        ov[o0 + q] = vals[a];
        if (oarg) oarg[o0 + q] = a;
    }
}

template <bool WRITE>
__global__ void __launch_bounds__(kPoolThreads)
pool_kernel(Geo g, PoolPlan p, const uint64_t* __restrict__ keys, const float* __restrict__ vals,
            const uint32_t* __restrict__ row_ptr, uint32_t* __restrict__ item_cnt,
            const uint64_t* __restrict__ item_off, uint64_t* __restrict__ ok, float* __restrict__ ov,
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
    const int64_t seg = r / p.PX;
    const int z0 = zc * p.zchunk;
    const int nz = min(p.zchunk, p.PZ - z0);
    for (int i = lane; i < nz; i += 32) {
        best[i] = 0u;
        arg[i] = 0xffffffffu;
    }
    __syncwarp();
    const int xa = px * p.sx, xb = min(xa + p.sx, g.X);
    const int ya = py * p.sy, yb = min(ya + p.sy, g.Y);
    // pass 1: max per cluster (or occupancy only when counting)
    for (int x = xa; x < xb; ++x) {
        for (int y = ya; y < yb; ++y) {
            const int64_t row = (seg * g.X + x) * (int64_t)g.Y + y;
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
    for (int x = xa; x < xb; ++x) {
        for (int y = ya; y < yb; ++y) {
            const int64_t row = (seg * g.X + x) * (int64_t)g.Y + y;
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
    const uint64_t pbase = ((uint64_t)(seg * p.PX + px) * p.PY + py) * (uint64_t)p.PZ + z0;
    for (int i0 = 0; i0 < nz; i0 += 32) {
        const int i = i0 + lane;
        const bool occ = i < nz && best[i] != 0u;
        const unsigned m = __ballot_sync(kFull, occ);
        if (occ) {
            const uint64_t o = pos + __popc(m & ((1u << lane) - 1u));
            const uint32_t a = arg[i];
            ok[o] = pbase + i;
            ov[o] = vals[a];
            if (oarg) oarg[o] = a;
        }
        pos += __popc(m);
    }
}

cudaError_t launch_maxpool(const Geo& g, const PoolPlan& p, const uint64_t* keys, const float* vals,
                           const uint32_t* row_ptr, uint32_t* item_cnt, uint64_t* item_off, uint64_t* scan_tmp,
                           uint64_t* out_keys, float* out_vals, int64_t* out_arg, int64_t* out_nnz, cudaStream_t s) {
    if (p.items == 0) return cudaMemsetAsync(out_nnz, 0, sizeof(int64_t), s);
    if (p.tiled) {
        const unsigned tg = (unsigned)p.items;
        { SPC_PHASE("pool_count", s, 1); pool_tile_kernel<false><<<tg, kTileThreads, 0, s>>>(g, p, keys, vals, row_ptr, item_cnt, nullptr, nullptr, nullptr, nullptr); }
        cudaError_t e = launch_scan_u32(item_cnt, item_off, p.items, out_nnz, scan_tmp, s);
        if (e != cudaSuccess) return e;
        { SPC_PHASE("pool_write", s, 1); pool_tile_kernel<true><<<tg, kTileThreads, 0, s>>>(g, p, keys, vals, row_ptr, item_cnt, item_off, out_keys, out_vals, out_arg); }
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

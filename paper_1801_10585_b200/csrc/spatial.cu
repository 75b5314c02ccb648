// Spatial sharding of one sample across GPUs (beyond the paper: P:90 keeps a
// whole grid on one GPU). The first spatial dimension is cut into contiguous plane ranges; a rank
// owns the outputs of its planes and needs the inputs of its planes +- the filter half-width
// (halo). Four device steps are exported here; the orchestration (halo exchange over NCCL, the
// per-round all-reduce of the selection histograms) is in spatial.py.
//
//   spc_slab_gather      per (b, c) segment, concatenate plane ranges of up to 4 source maps and
//                        re-base them into a grid with another plane count (halo assembly, owned-
//                        plane extraction, shard <-> global keys); optional source index.
//   spc_topk_digit_hist  one 8-bit digit histogram per segment of the attention composite
//                        (score << 32 | ~p_global, reading R7) among the entries matching the
//                        prefix chosen so far -- summed over ranks by the caller.
//   spc_topk_digit_pick  per segment, the digit holding the k-th largest composite of the summed
//                        histogram; after 8 rounds the prefix IS the k-th composite.
//   spc_topk_keep_ge     keep the entries whose composite >= that threshold, in key order.
//   spc_index_add        out[idx[t]] += v[t] (halo partials of dx returned to their owner).
#include "spc_internal.cuh"
#include "block_scan.cuh"

#include <algorithm>

using namespace spc;

namespace {

constexpr int kMaxSrc = 4;

struct GatherSrc {
    const uint64_t* keys;
    const float* values;
    const int64_t* n_dev;
    int64_t n;
    int64_t planes;      // plane count of the source grid
    int64_t lo, hi;      // kept planes [lo, hi) (source coordinates)
    int64_t shift;       // output plane = source plane + shift
    int64_t base;        // first index of this source in the concatenated source index space
};
struct GatherArgs {
    GatherSrc src[kMaxSrc];
    int nsrc;
    int64_t nseg;
    uint64_t plane;      // entries per plane (product of the other spatial dims)
    int64_t planes_out;
};

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* k, int64_t n, uint64_t want) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t m = (lo + hi) >> 1;
        if (k[m] < want) lo = m + 1;
        else hi = m;
    }
    return lo;
}

// piece = seg * nsrc + j: start[piece] (source entry), cnt[piece]
__global__ void gather_bounds_kernel(GatherArgs a, int64_t* __restrict__ start, int64_t* __restrict__ cnt) {
    const int64_t piece = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (piece >= a.nseg * a.nsrc) return;
    const int j = (int)(piece % a.nsrc);
    const int64_t seg = piece / a.nsrc;
    const GatherSrc& s = a.src[j];
    const int64_t n = load_n(s.n_dev, s.n);
    const uint64_t seg0 = (uint64_t)seg * (uint64_t)s.planes * a.plane;
    const int64_t b = lower_bound_u64(s.keys, n, seg0 + (uint64_t)s.lo * a.plane);
    const int64_t e = lower_bound_u64(s.keys, n, seg0 + (uint64_t)s.hi * a.plane);
    start[piece] = b;
    cnt[piece] = e - b;
}

// Exclusive scan of cnt[0..m) into off[0..m], off[m] = total -> *nnz_dev. One block.
__global__ void gather_scan_kernel(const int64_t* __restrict__ cnt, int64_t m, int64_t* __restrict__ off,
                                   int64_t* __restrict__ nnz_dev) {
    __shared__ int64_t carry;
    __shared__ int64_t warp_tot[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t c0 = 0; c0 < m; c0 += blockDim.x) {
        const int64_t i = c0 + threadIdx.x;
        const int64_t v = i < m ? cnt[i] : 0;
        int64_t x = v;
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) warp_tot[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int64_t t = lane < nw ? warp_tot[lane] : 0;
            for (int d = 1; d < 32; d <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, t, d);
                if (lane >= d) t += y;
            }
            if (lane < nw) warp_tot[lane] = t;   // inclusive over warps
        }
        __syncthreads();
        const int64_t before = carry + (wid ? warp_tot[wid - 1] : 0);
        if (i < m) off[i] = before + x - v;
        __syncthreads();
        if (threadIdx.x == 0) carry += warp_tot[nw - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        off[m] = carry;
        *nnz_dev = carry;
    }
}

// Output entry i -> its piece by binary search over off[] (pieces are few), then one copy with the
// key re-based: out = key + seg * (planes_out - planes_src) * plane + shift * plane.
__global__ void gather_write_kernel(GatherArgs a, const int64_t* __restrict__ start, const int64_t* __restrict__ off,
                                    int64_t bound, uint64_t* __restrict__ okeys, float* __restrict__ ovals,
                                    int64_t* __restrict__ src_index) {
    const int64_t m = a.nseg * a.nsrc;
    const int64_t total = min(off[m], bound);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = m;   // last piece with off[piece] <= i
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (off[mid] <= i) lo = mid;
            else hi = mid;
        }
        const int64_t piece = lo;
        const int j = (int)(piece % a.nsrc);
        const int64_t seg = piece / a.nsrc;
        const GatherSrc& s = a.src[j];
        const int64_t e = start[piece] + (i - off[piece]);
        const uint64_t k = s.keys[e];
        okeys[i] = k + (uint64_t)((int64_t)seg * (a.planes_out - s.planes) * (int64_t)a.plane + s.shift * (int64_t)a.plane);
        ovals[i] = s.values[e];
        if (src_index) src_index[i] = s.base + e;
    }
}

__device__ __forceinline__ uint64_t composite_of(uint64_t key, float v, uint64_t V, uint64_t p_base, int attn) {
    const uint64_t p = key % V + p_base;
    return ((uint64_t)score_bits(__float_as_uint(v), attn) << 32) | (uint64_t)(~(uint32_t)p);
}

// Digit histogram: bits [shift, shift + 8) of the composite among the entries whose higher bits
// equal prefix[seg]'s; segments with need[seg] < 0 are settled and skipped. Blocks take chunks of
// consecutive entries; a chunk spanning at most 4 segments (the usual case: segments are long)
// finds an entry's segment by comparing with the chunk's segment bounds (no 64-bit division) and
// counts in shared bins, aggregated per warp over lanes with the same (segment, digit) -- round 1
// sees few distinct digits (the exponent byte), so plain atomics would serialise on them.
constexpr int kHistChunk = 4096;
__global__ void digit_hist_kernel(const uint64_t* __restrict__ keys, const float* __restrict__ vals,
                                  const int64_t* nnz_dev, int64_t bound, uint64_t V, uint64_t p_base, int attn,
                                  const uint64_t* __restrict__ prefix, const int64_t* __restrict__ need, int shift,
                                  uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[4 * 256];
    __shared__ int64_t s_need[4];
    __shared__ uint64_t s_pre[4];
    const int64_t n = load_n(nnz_dev, bound);
    const int lane = threadIdx.x & 31;
    for (int64_t c0 = (int64_t)blockIdx.x * kHistChunk; c0 < n; c0 += (int64_t)gridDim.x * kHistChunk) {
        const int64_t c1 = min(c0 + kHistChunk, n);
        const int64_t s0 = (int64_t)(keys[c0] / V);
        const int64_t s1 = (int64_t)(keys[c1 - 1] / V);
        const bool local = s1 - s0 < 4;
        if (local) {
            for (int t = threadIdx.x; t < 4 * 256; t += blockDim.x) sh[t] = 0;
            if (threadIdx.x < 4 && s0 + threadIdx.x <= s1) {
                s_need[threadIdx.x] = need[s0 + threadIdx.x];
                s_pre[threadIdx.x] = prefix[s0 + threadIdx.x];
            }
            __syncthreads();
            const uint64_t base0 = (uint64_t)s0 * V;
            // whole warps step together (the aggregation needs converged lanes)
            for (int64_t i0 = c0 + (threadIdx.x & ~31); i0 < c1; i0 += blockDim.x) {
                const int64_t i = i0 + lane;
                int slot = -1;
                uint32_t d = 0;
                if (i < c1) {
                    const uint64_t k = keys[i];
                    uint64_t rel = k - base0;
                    int si = 0;
                    while (rel >= V) {
                        rel -= V;
                        ++si;
                    }
                    if (s_need[si] >= 0) {
                        const uint64_t c = ((uint64_t)score_bits(__float_as_uint(vals[i]), attn) << 32) |
                                           (uint64_t)(~(uint32_t)(rel + p_base));
                        if (shift >= 56 || (c >> (shift + 8)) == (s_pre[si] >> (shift + 8))) {
                            d = (uint32_t)(c >> shift) & 255u;
                            slot = si * 256 + (int)d;
                        }
                    }
                }
                const unsigned act = __ballot_sync(0xffffffffu, slot >= 0);
                if (slot >= 0) {
                    const unsigned same = __match_any_sync(act, slot);
                    if (lane == __ffs(same) - 1) atomicAdd(&sh[slot], (uint32_t)__popc(same));
                }
            }
            __syncthreads();
            for (int t = threadIdx.x; t < (int)(s1 - s0 + 1) * 256; t += blockDim.x)
                if (sh[t]) atomicAdd(&hist[(s0 + t / 256) * 256 + (t & 255)], sh[t]);
            __syncthreads();
        } else {
            for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
                const uint64_t k = keys[i];
                const int64_t seg = (int64_t)(k / V);
                if (need[seg] < 0) continue;
                const uint64_t c = composite_of(k, vals[i], V, p_base, attn);
                if (shift < 56 && (c >> (shift + 8)) != (prefix[seg] >> (shift + 8))) continue;
                atomicAdd(&hist[seg * 256 + ((uint32_t)(c >> shift) & 255u)], 1u);
            }
        }
    }
}

// One block of 256 threads per segment: suffix counts from the top digit, pick d with
// above(d) < need <= above(d) + hist[d]. First round: a segment with at most k entries in total
// keeps all of them (threshold 0, need = -1: settled).
__global__ void digit_pick_kernel(int64_t nseg, const uint32_t* __restrict__ hist, int shift,
                                  uint64_t* __restrict__ prefix, int64_t* __restrict__ need) {
    __shared__ int64_t suf[257];
    const int64_t seg = blockIdx.x;
    if (seg >= nseg) return;
    const int64_t nd = need[seg];
    if (nd < 0) return;
    const int t = threadIdx.x;
    if (t == 0) {   // serial suffix sum of 256 bins (tiny)
        int64_t acc = 0;
        suf[256] = 0;
        for (int d = 255; d >= 0; --d) {
            acc += hist[seg * 256 + d];
            suf[d] = acc;
        }
    }
    __syncthreads();
    if (shift == 56 && suf[0] <= nd) {
        if (t == 0) {
            prefix[seg] = 0;
            need[seg] = -1;
        }
        return;
    }
    // exactly one d satisfies suf[d + 1] < nd <= suf[d]
    if (suf[t + 1] < nd && nd <= suf[t]) {
        prefix[seg] |= (uint64_t)t << shift;
        const int64_t rest = nd - suf[t + 1];
        // the whole bucket is kept: prefix (lower bits 0) is already an exact threshold
        need[seg] = rest == suf[t] - suf[t + 1] ? -1 : rest;
    }
}

// Keep composite >= thr[seg], order preserved: per-tile counts, one-block scan, write. A tile
// spanning at most 4 segments finds an entry's segment by comparing with the tile's segment
// bounds (no 64-bit division per entry).
struct TileSegs {
    int64_t s0;
    int span;            // s1 - s0 + 1 when <= 4, else 0 (divide per entry)
    uint64_t thr[4];
};
__device__ __forceinline__ void tile_segs(TileSegs& t, const uint64_t* keys, int64_t c0, int64_t c1, uint64_t V,
                                          const uint64_t* thr) {
    if (threadIdx.x == 0) {
        t.s0 = (int64_t)(keys[c0] / V);
        const int64_t s1 = (int64_t)(keys[c1 - 1] / V);
        t.span = s1 - t.s0 < 4 ? (int)(s1 - t.s0 + 1) : 0;
        for (int j = 0; j < t.span; ++j) t.thr[j] = thr[t.s0 + j];
    }
}
__device__ __forceinline__ bool keep_entry(const TileSegs& t, uint64_t k, float v, uint64_t V, uint64_t p_base,
                                           int attn, const uint64_t* thr) {
    uint64_t rel, th;
    if (t.span) {
        rel = k - (uint64_t)t.s0 * V;
        int si = 0;
        while (rel >= V) {
            rel -= V;
            ++si;
        }
        th = t.thr[si];
    } else {
        const uint64_t seg = k / V;
        rel = k - seg * V;
        th = thr[seg];
    }
    const uint64_t c = ((uint64_t)score_bits(__float_as_uint(v), attn) << 32) | (uint64_t)(~(uint32_t)(rel + p_base));
    return c >= th;
}

constexpr int kKeepTile = 2048;
__global__ void keep_count_kernel(const uint64_t* __restrict__ keys, const float* __restrict__ vals,
                                  const int64_t* nnz_dev, int64_t bound, uint64_t V, uint64_t p_base, int attn,
                                  const uint64_t* __restrict__ thr, int64_t* __restrict__ tile_cnt, int64_t ntiles) {
    __shared__ int cnt;
    __shared__ TileSegs ts;
    const int64_t n = load_n(nnz_dev, bound);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t c0 = tile * kKeepTile, c1 = min(c0 + kKeepTile, n);
        if (threadIdx.x == 0) cnt = 0;
        if (c0 < c1) tile_segs(ts, keys, c0, c1, V, thr);
        __syncthreads();
        int mine = 0;
        for (int64_t i = c0 + threadIdx.x; i < c1; i += blockDim.x)
            mine += keep_entry(ts, keys[i], vals[i], V, p_base, attn, thr);
        for (int d = 16; d; d >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, d);
        if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&cnt, mine);
        __syncthreads();
        if (threadIdx.x == 0) tile_cnt[tile] = cnt;
        __syncthreads();
    }
}

__global__ void keep_write_kernel(const uint64_t* __restrict__ keys, const float* __restrict__ vals,
                                  const int64_t* nnz_dev, int64_t bound, uint64_t V, uint64_t p_base, int attn,
                                  const uint64_t* __restrict__ thr, const int64_t* __restrict__ tile_off, int64_t ntiles,
                                  uint64_t* __restrict__ okeys, float* __restrict__ ovals, int64_t* __restrict__ src_index) {
    __shared__ int warp_cnt[32];
    __shared__ int64_t base;
    __shared__ TileSegs ts;
    const int64_t n = load_n(nnz_dev, bound);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t c0 = tile * kKeepTile, c1 = min(c0 + kKeepTile, n);
        if (threadIdx.x == 0) base = tile_off[tile];
        if (c0 < c1) tile_segs(ts, keys, c0, c1, V, thr);
        __syncthreads();
        for (int64_t r0 = c0; r0 < c1; r0 += blockDim.x) {   // rounds of blockDim entries, in order
            const int64_t i = r0 + threadIdx.x;
            bool keep = false;
            uint64_t k = 0;
            float v = 0.f;
            if (i < c1) {
                k = keys[i];
                v = vals[i];
                keep = keep_entry(ts, k, v, V, p_base, attn, thr);
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) warp_cnt[wid] = __popc(m);
            __syncthreads();
            int before = 0, round_tot = 0;
            for (int w = 0; w < nw; ++w) {
                before += w < wid ? warp_cnt[w] : 0;
                round_tot += warp_cnt[w];
            }
            if (keep) {
                const int64_t o = base + before + __popc(m & ((1u << lane) - 1u));
                okeys[o] = k;
                ovals[o] = v;
                if (src_index) src_index[o] = i;
            }
            __syncthreads();
            if (threadIdx.x == 0) base += round_tot;
            __syncthreads();
        }
    }
}

__global__ void index_add_kernel(const int64_t* __restrict__ idx, const float* __restrict__ v, const int64_t* n_dev,
                                 int64_t bound, float* __restrict__ out) {
    const int64_t n = load_n(n_dev, bound);
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
        out[idx[t]] += v[t];
}

spc_status_t cu(cudaError_t e) { return e == cudaSuccess ? SPC_OK : SPC_ERR_CUDA; }

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

bool plain64(const spc_map_t* m) { return m->key_bits == 0 || m->key_bits == 64; }

spc_status_t check_sel_map(const spc_map_t* x, int64_t p_base, uint64_t* V) {
    if (!x || x->ndim < 1 || x->ndim > SPC_MAX_NDIM || x->batch < 0 || x->channels < 1 || x->nnz < 0)
        return SPC_ERR_INVALID_ARG;
    if (!plain64(x)) return SPC_ERR_UNSUPPORTED;
    if (x->nnz > 0 && (!x->keys || !x->values)) return SPC_ERR_INVALID_ARG;
    double v = 1;
    for (int d = 0; d < x->ndim; ++d) {
        if (x->dims[d] < 1) return SPC_ERR_SHAPE;
        v *= (double)x->dims[d];
    }
    if (p_base < 0 || v + (double)p_base > 4294967296.0) return SPC_ERR_UNSUPPORTED;   // composite needs p < 2^32
    *V = (uint64_t)v;
    return SPC_OK;
}

}  // namespace

extern "C" spc_status_t spc_slab_gather_query(int64_t nseg, int32_t nsrc, size_t* workspace_bytes) {
    if (!workspace_bytes || nseg < 0 || nsrc < 1 || nsrc > kMaxSrc) return SPC_ERR_INVALID_ARG;
    const int64_t m = nseg * nsrc;
    *workspace_bytes = align256((size_t)m * 8) + align256((size_t)(m + 1) * 8) + align256((size_t)m * 8);
    return SPC_OK;
}

extern "C" spc_status_t spc_slab_gather(const spc_slab_src_t* srcs, int32_t nsrc, int64_t nseg, int64_t plane,
                                        int64_t planes_out, spc_map_out_t* y, int64_t* src_index, void* workspace,
                                        size_t workspace_bytes, cudaStream_t s) {
    if (!srcs || nsrc < 1 || nsrc > kMaxSrc || nseg < 0 || plane < 1 || planes_out < 1 || !y || !y->nnz_dev)
        return SPC_ERR_INVALID_ARG;
    if (y->key_bits != 0 && y->key_bits != 64) return SPC_ERR_UNSUPPORTED;
    size_t need = 0;
    spc_slab_gather_query(nseg, nsrc, &need);
    if (workspace_bytes < need || (need && !workspace)) return SPC_ERR_WORKSPACE;
    if ((double)nseg * (double)planes_out * (double)plane >= 1.8e19) return SPC_ERR_SHAPE;
    GatherArgs a{};
    a.nsrc = nsrc;
    a.nseg = nseg;
    a.plane = (uint64_t)plane;
    a.planes_out = planes_out;
    int64_t bound = 0;
    for (int j = 0; j < nsrc; ++j) {
        const spc_slab_src_t& q = srcs[j];
        if (q.n < 0 || q.planes < 1 || q.lo < 0 || q.hi < q.lo || q.hi > q.planes) return SPC_ERR_INVALID_ARG;
        if (q.n > 0 && (!q.keys || !q.values)) return SPC_ERR_INVALID_ARG;
        if (q.hi > q.lo && (q.lo + q.shift < 0 || q.hi + q.shift > planes_out)) return SPC_ERR_SHAPE;
        a.src[j] = GatherSrc{q.keys, q.values, q.nnz_dev, q.n, q.planes, q.lo, q.hi, q.shift, bound};
        bound += q.n;
    }
    if (y->capacity < bound || (bound > 0 && (!y->keys || !y->values))) return SPC_ERR_CAPACITY;
    const int64_t m = nseg * nsrc;
    char* w = (char*)workspace;
    int64_t* start = (int64_t*)w;
    int64_t* off = (int64_t*)(w + align256((size_t)m * 8));
    int64_t* cnt = (int64_t*)(w + align256((size_t)m * 8) + align256((size_t)(m + 1) * 8));
    SPC_PHASE("slab_gather", s, m > 0 ? 3 : 1);
    if (m == 0) return cu(cudaMemsetAsync(y->nnz_dev, 0, sizeof(int64_t), s));
    gather_bounds_kernel<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(a, start, cnt);
    gather_scan_kernel<<<1, 1024, 0, s>>>(cnt, m, off, y->nnz_dev);
    if (bound > 0) {
        const unsigned grid = (unsigned)std::min<int64_t>((bound + 255) / 256, (int64_t)num_sms() * 8);
        gather_write_kernel<<<grid, 256, 0, s>>>(a, start, off, bound, y->keys, y->values, src_index);
    }
    return cu(cudaGetLastError());
}

extern "C" spc_status_t spc_topk_digit_hist(const spc_map_t* x, spc_attn_t attn, int64_t p_base, const uint64_t* prefix,
                                            const int64_t* need, int32_t shift, uint32_t* hist, cudaStream_t s) {
    uint64_t V = 0;
    if (spc_status_t e = check_sel_map(x, p_base, &V)) return e;
    if (attn != SPC_ATTN_MAGNITUDE && attn != SPC_ATTN_RAW) return SPC_ERR_INVALID_ARG;
    if (shift < 0 || shift > 56 || shift % 8 || !prefix || !need || !hist) return SPC_ERR_INVALID_ARG;
    SPC_PHASE("topk_digit_hist", s, 1);
    if (x->nnz == 0) return SPC_OK;
    const int64_t chunks = (x->nnz + kHistChunk - 1) / kHistChunk;
    const unsigned grid = (unsigned)std::min<int64_t>(chunks, (int64_t)num_sms() * 8);
    digit_hist_kernel<<<grid, 256, 0, s>>>(x->keys, x->values, x->nnz_dev, x->nnz, V, (uint64_t)p_base, (int)attn,
                                           prefix, need, shift, hist);
    return cu(cudaGetLastError());
}

extern "C" spc_status_t spc_topk_digit_pick(int64_t nseg, const uint32_t* hist, int32_t shift, uint64_t* prefix,
                                            int64_t* need, cudaStream_t s) {
    if (nseg < 0 || shift < 0 || shift > 56 || shift % 8) return SPC_ERR_INVALID_ARG;
    if (nseg > 0 && (!hist || !prefix || !need)) return SPC_ERR_INVALID_ARG;
    SPC_PHASE("topk_digit_pick", s, 1);
    if (nseg == 0) return SPC_OK;
    digit_pick_kernel<<<(unsigned)nseg, 256, 0, s>>>(nseg, hist, shift, prefix, need);
    return cu(cudaGetLastError());
}

extern "C" spc_status_t spc_topk_keep_query(const spc_map_t* x, size_t* workspace_bytes) {
    if (!x || !workspace_bytes || x->nnz < 0) return SPC_ERR_INVALID_ARG;
    const int64_t ntiles = (x->nnz + kKeepTile - 1) / kKeepTile;
    *workspace_bytes = align256((size_t)(ntiles + 1) * 8) * 2;
    return SPC_OK;
}

extern "C" spc_status_t spc_topk_keep_ge(const spc_map_t* x, spc_attn_t attn, int64_t p_base, const uint64_t* thr,
                                         spc_map_out_t* y, int64_t* src_index, void* workspace, size_t workspace_bytes,
                                         cudaStream_t s) {
    uint64_t V = 0;
    if (spc_status_t e = check_sel_map(x, p_base, &V)) return e;
    if (attn != SPC_ATTN_MAGNITUDE && attn != SPC_ATTN_RAW) return SPC_ERR_INVALID_ARG;
    if (!y || !y->nnz_dev || !thr) return SPC_ERR_INVALID_ARG;
    if (y->key_bits != 0 && y->key_bits != 64) return SPC_ERR_UNSUPPORTED;
    if (y->capacity < x->nnz || (x->nnz > 0 && (!y->keys || !y->values))) return SPC_ERR_CAPACITY;
    size_t need = 0;
    spc_topk_keep_query(x, &need);
    if (workspace_bytes < need || !workspace) return SPC_ERR_WORKSPACE;
    const int64_t ntiles = (x->nnz + kKeepTile - 1) / kKeepTile;
    int64_t* tile_cnt = (int64_t*)workspace;
    int64_t* tile_off = (int64_t*)((char*)workspace + align256((size_t)(ntiles + 1) * 8));
    SPC_PHASE("topk_keep_ge", s, ntiles ? 3 : 1);
    if (ntiles == 0) return cu(cudaMemsetAsync(y->nnz_dev, 0, sizeof(int64_t), s));
    const unsigned grid = (unsigned)std::min<int64_t>(ntiles, (int64_t)num_sms() * 8);
    keep_count_kernel<<<grid, 256, 0, s>>>(x->keys, x->values, x->nnz_dev, x->nnz, V, (uint64_t)p_base, (int)attn,
                                           thr, tile_cnt, ntiles);
    gather_scan_kernel<<<1, 1024, 0, s>>>(tile_cnt, ntiles, tile_off, y->nnz_dev);
    keep_write_kernel<<<grid, 256, 0, s>>>(x->keys, x->values, x->nnz_dev, x->nnz, V, (uint64_t)p_base, (int)attn, thr,
                                           tile_off, ntiles, y->keys, y->values, src_index);
    return cu(cudaGetLastError());
}

extern "C" spc_status_t spc_index_add(const int64_t* idx, const float* v, int64_t n_bound, const int64_t* n_dev,
                                      float* out, cudaStream_t s) {
    if (n_bound < 0 || (n_bound > 0 && (!idx || !v || !out))) return SPC_ERR_INVALID_ARG;
    SPC_PHASE("index_add", s, 1);
    if (n_bound == 0) return SPC_OK;
    const unsigned grid = (unsigned)std::min<int64_t>((n_bound + 255) / 256, (int64_t)num_sms() * 8);
    index_add_kernel<<<grid, 256, 0, s>>>(idx, v, n_dev, n_bound, out);
    return cu(cudaGetLastError());
}

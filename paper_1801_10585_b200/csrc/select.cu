// Attention as a standalone layer: per (b, c) segment of a COO map keep the k
// entries with the largest score (|y| for variant (ii), y for variant (i)); ties go to the
// smaller key (reading R7). The fused forward has its own pipeline (conv_fwd.cu, fwd_stream.cu);
// this one serves attention_topk.
//
// Streamed over tiles of kTkTile entries (a tile never spans two segments), so every pass runs
// on the whole GPU whatever the number and size of the segments:
//   plan:    per segment its kept count min(n, k) -> output offsets, and its first tile;
//   hist:    per tile a histogram of the top score digit (13 bits when the segments are large
//            enough to amortise 8192 bins, else 11), added to the segment's;
//   find:    per segment the digit B1 holding the k-th largest score; the whole bucket is kept
//            when it holds exactly the entries still needed (mode 1), else it is resolved
//            exactly (mode 2); segments with n <= k keep everything (mode 0);
//   collect: per tile the entries above B1 are counted, those in B1 (mode 2) appended to the
//            segment's candidate list as composite keys (score << 32 | ~local index);
//   select:  per segment the need-th largest candidate (radix select) -> kstar; per tile the
//            selected candidates are counted and the segment's tiles get their output offsets;
//   write:   per tile an ordered compaction of the kept entries (keys, values, sources).
// The values are read three times (hist, collect, write) and the keys once.
#include "spc_internal.cuh"
#include "block_scan.cuh"

#include <algorithm>

namespace spc {

constexpr int kTkTile = 4096;                         // entries per tile
constexpr int kTkThreads = 256;
constexpr int kTkItems = kTkTile / kTkThreads;        // 16 entries per thread
constexpr uint32_t kTkSmemCand = 12288;               // candidates selected in shared memory (96 KB, dynamic)

struct TkSeg {
    uint64_t kstar;    // mode 2: keep composite >= kstar within bucket b1
    uint32_t b1;       // threshold digit (score >> (32 - bits))
    uint32_t mode;     // 0 keep all, 1 keep digit >= b1, 2 keep digit > b1 or composite >= kstar
    uint32_t need;     // mode 2: entries to take from bucket b1
    uint32_t pad;
};

size_t topk_tiles_bound(int64_t nnz, int64_t nseg) { return (size_t)(nnz / kTkTile + nseg + 1); }
size_t topk_seg_bytes() { return sizeof(TkSeg); }
constexpr int kTkMaxBins = 8192;
// 13-bit first digit (1/16 of the 11-bit bucket: fewer candidates, a shorter select) when the
// per-segment histograms stay small next to the data (>= 32 Ki entries per segment on average)
int topk_bits(int64_t nnz, int64_t nseg) { return nseg * (int64_t)kTkMaxBins * 4 <= nnz ? 13 : 11; }

__device__ __forceinline__ uint64_t tk_comp(uint32_t sc, uint32_t local) {
    return ((uint64_t)sc << 32) | (uint64_t)(0xffffffffu - local);
}

// tile -> segment map (one dependent load for a tile kernel instead of a binary search)
__global__ void topk_tile_map_kernel(const uint32_t* __restrict__ tile_start, int64_t nseg,
                                     uint32_t* __restrict__ tile_seg) {
    for (int64_t s = blockIdx.x; s < nseg; s += gridDim.x)
        for (uint32_t t = tile_start[s] + threadIdx.x; t < tile_start[s + 1]; t += blockDim.x) tile_seg[t] = (uint32_t)s;
}

// seg_off[s] = sum over earlier segments of min(n_s', k); tile_start[s] = sum of ceil(n_s' / tile)
__global__ void topk_plan_kernel(const uint32_t* __restrict__ seg_lo, int64_t nseg, int64_t k,
                                 uint64_t* __restrict__ seg_off, uint32_t* __restrict__ tile_start,
                                 int64_t* __restrict__ total) {
    __shared__ uint64_t sm[33];
    uint64_t carry = 0, tcarry = 0;
    for (int64_t base = 0; base < nseg; base += blockDim.x) {
        const int64_t s = base + threadIdx.x;
        uint64_t v = 0, nt = 0;
        if (s < nseg) {
            const uint64_t n = (uint64_t)(seg_lo[s + 1] - seg_lo[s]);
            v = n <= (uint64_t)k ? n : (uint64_t)k;
            nt = (n + kTkTile - 1) / kTkTile;
        }
        uint64_t t;
        const uint64_t packed = (v << 24) | nt;   // (kept < 2^32 per call, tiles < 2^24)
        const uint64_t ex = block_excl_scan(packed, sm, &t);
        if (s < nseg) {
            seg_off[s] = carry + (ex >> 24);
            tile_start[s] = (uint32_t)(tcarry + (ex & 0xffffffull));
        }
        carry += t >> 24;
        tcarry += t & 0xffffffull;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *total = (int64_t)carry;
        tile_start[nseg] = (uint32_t)tcarry;
    }
}

struct TkTile {
    int64_t s;
    uint32_t lo, hi;   // entries [lo, hi) of the tile
    uint32_t seg0;     // first entry of the segment
    bool ok;
};
__device__ __forceinline__ TkTile tk_tile(const uint32_t* seg_lo, const uint32_t* tile_start, const uint32_t* tile_seg,
                                          int64_t nseg, uint32_t t) {
    TkTile r{};
    r.ok = t < __ldg(&tile_start[nseg]);
    if (!r.ok) return r;
    r.s = __ldg(&tile_seg[t]);
    r.seg0 = __ldg(&seg_lo[r.s]);
    r.lo = r.seg0 + (t - __ldg(&tile_start[r.s])) * (uint32_t)kTkTile;
    r.hi = min(r.lo + (uint32_t)kTkTile, __ldg(&seg_lo[r.s + 1]));
    return r;
}

// A block takes kTkHistTiles consecutive tiles (the histogram's zeroing and flush amortised over
// them), flushing into the segment's histogram whenever the segment changes; the next tile's
// loads are issued before the current one's bins are updated.
constexpr int kTkHistTiles = 4;
template <int ATTN>
__global__ void __launch_bounds__(kTkThreads) topk_hist_kernel(const float* __restrict__ vals,
                                                               const uint32_t* __restrict__ seg_lo,
                                                               const uint32_t* __restrict__ tile_start,
                                                               const uint32_t* __restrict__ tile_seg, int64_t nseg,
                                                               int attn, int64_t k, int bits,
                                                               uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kTkMaxBins];
    const int nb = 1 << bits, sh = 32 - bits;
    for (int i = threadIdx.x; i < nb; i += kTkThreads) h[i] = 0u;
    int64_t cur = -1;   // segment whose counts the shared histogram holds
    auto flush = [&]() {
        __syncthreads();
        uint32_t* gh = hist + (cur << bits);
        for (int i = threadIdx.x; i < nb; i += kTkThreads) {
            const uint32_t v = h[i];
            if (v) {
                atomicAdd(&gh[i], v);
                h[i] = 0u;
            }
        }
        __syncthreads();
    };
    const uint32_t t0 = blockIdx.x * kTkHistTiles;
    uint32_t b[kTkItems];
    TkTile tl = tk_tile(seg_lo, tile_start, tile_seg, nseg, t0);
    auto load = [&](const TkTile& q, bool keep_all) {
#pragma unroll
        for (int u = 0; u < kTkItems; ++u) {
            const uint32_t i = q.lo + (uint32_t)(u * kTkThreads) + threadIdx.x;
            b[u] = (!keep_all && i < q.hi) ? __float_as_uint(__ldg(&vals[i])) : 0u;
        }
    };
    bool ka = tl.ok && (int64_t)(__ldg(&seg_lo[tl.s + 1]) - tl.seg0) <= k;   // keep-all segment: no histogram
    if (tl.ok) load(tl, ka);
    __syncthreads();
    for (int tt = 0; tt < kTkHistTiles && tl.ok; ++tt) {
        if (!ka && tl.s != cur) {
            if (cur >= 0) flush();
            cur = tl.s;
        }
        uint32_t sc[kTkItems];
#pragma unroll
        for (int u = 0; u < kTkItems; ++u) sc[u] = score_bits(b[u], ATTN);
        const TkTile cu = tl;
        const bool cka = ka;
        if (tt + 1 < kTkHistTiles) {   // next tile's loads in flight
            tl = tk_tile(seg_lo, tile_start, tile_seg, nseg, t0 + tt + 1);
            ka = tl.ok && (int64_t)(__ldg(&seg_lo[tl.s + 1]) - tl.seg0) <= k;
            if (tl.ok) load(tl, ka);
        } else {
            tl.ok = false;
        }
        if (!cka) {
#pragma unroll
            for (int u = 0; u < kTkItems; ++u) {
                const uint32_t i = cu.lo + (uint32_t)(u * kTkThreads) + threadIdx.x;
                if (i < cu.hi) atomicAdd(&h[sc[u] >> sh], 1u);
            }
        }
    }
    if (cur >= 0) flush();
}

__global__ void topk_find_kernel(const uint32_t* __restrict__ seg_lo, int64_t k, int bits,
                                 const uint32_t* __restrict__ hist, TkSeg* __restrict__ seg,
                                 uint32_t* __restrict__ cand_cnt) {
    __shared__ uint32_t sm[33];
    const int64_t s = blockIdx.x;
    const uint64_t n = (uint64_t)(seg_lo[s + 1] - seg_lo[s]);
    if (n <= (uint64_t)k) {
        if (threadIdx.x == 0) {
            TkSeg st{};
            st.mode = 0;
            seg[s] = st;
            cand_cnt[s] = 0;
        }
        return;
    }
    const int nb = 1 << bits;
    __shared__ uint32_t h[kTkMaxBins];   // the segment's histogram, staged with coalesced loads
    for (int i = threadIdx.x; i < nb; i += blockDim.x) h[i] = hist[(s << bits) + i];
    __syncthreads();
    const int per = nb / 256;   // blockDim 256: bins from the top, per thread a stripe
    uint32_t own = 0;
    for (int q = 0; q < per; ++q)   // (rotated start: the 32 lanes' reads hit distinct banks)
        own += h[nb - 1 - threadIdx.x * per - ((q + (int)threadIdx.x) & (per - 1))];
    uint32_t tot;
    const uint32_t before = block_excl_scan(own, sm, &tot);
    if (before < (uint32_t)k && before + own >= (uint32_t)k) {
        uint32_t cum = before;
        for (int q = 0; q < per; ++q) {
            const int bin = nb - 1 - threadIdx.x * per - q;
            if (cum + h[bin] >= (uint32_t)k) {
                TkSeg st{};
                st.b1 = (uint32_t)bin;
                st.need = (uint32_t)k - cum;
                st.mode = st.need == h[bin] ? 1u : 2u;
                seg[s] = st;
                cand_cnt[s] = 0;
                break;
            }
            cum += h[bin];
        }
    }
}

template <int ATTN>
__global__ void __launch_bounds__(kTkThreads) topk_collect_kernel(const float* __restrict__ vals,
                                                                  const uint32_t* __restrict__ seg_lo,
                                                                  const uint32_t* __restrict__ tile_start,
                                                                  const uint32_t* __restrict__ tile_seg,
                                                                  int64_t nseg, int attn, int bits,
                                                                  const TkSeg* __restrict__ seg,
                                                                  uint64_t* __restrict__ cand,
                                                                  uint32_t* __restrict__ cand_cnt,
                                                                  uint32_t* __restrict__ tile_def) {
    __shared__ uint32_t sm[33];
    const TkTile tl = tk_tile(seg_lo, tile_start, tile_seg, nseg, blockIdx.x);
    if (!tl.ok) return;
    const TkSeg st = seg[tl.s];
    if (st.mode == 0) {
        if (threadIdx.x == 0) tile_def[blockIdx.x] = tl.hi - tl.lo;
        return;
    }
    uint32_t b[kTkItems];
#pragma unroll
    for (int u = 0; u < kTkItems; ++u) {
        const uint32_t i = tl.lo + (uint32_t)(u * kTkThreads) + threadIdx.x;
        b[u] = i < tl.hi ? __float_as_uint(__ldg(&vals[i])) : 0u;
    }
    // count first, one atomic per tile for the tile's slots in the segment's candidate list
    // (the list is unordered: the select does not care), then write
    // kept for sure: score >= ldef (digit above b1, or b1 itself in mode 1); candidates (mode
    // 2): score - cb < wb (digit b1). Scores are compared directly, no digit extraction.
    const int sh = 32 - bits;
    const uint64_t ldef64 = (uint64_t)(st.mode == 1u ? st.b1 : st.b1 + 1u) << sh;
    const bool none_above = ldef64 > 0xffffffffull;
    const uint32_t ldef = (uint32_t)ldef64, cb = st.b1 << sh, wb = st.mode == 2u ? 1u << sh : 0u;
    const uint32_t nin = tl.hi - tl.lo;
    uint32_t def = 0, nc = 0, cm = 0;
#pragma unroll
    for (int u = 0; u < kTkItems; ++u) {
        const bool in = (uint32_t)(u * kTkThreads) + threadIdx.x < nin;
        const uint32_t sc = score_bits(b[u], ATTN);
        def += (in && sc >= ldef && !none_above) ? 1u : 0u;
        const bool c = in && (sc - cb) < wb;
        cm |= (c ? 1u : 0u) << u;
        nc += c ? 1u : 0u;
    }
    __shared__ uint32_t sh_base;
    uint32_t ctot;
    const uint32_t cex = block_excl_scan(nc, sm, &ctot);
    if (threadIdx.x == 0 && ctot) sh_base = atomicAdd(&cand_cnt[tl.s], ctot);
    __syncthreads();
    if (cm) {
        uint64_t* cs = cand + tl.seg0 + sh_base + cex;   // the segment's candidates (at most its size)
#pragma unroll
        for (int u = 0; u < kTkItems; ++u)
            if ((cm >> u) & 1u) {
                const uint32_t i = tl.lo + (uint32_t)(u * kTkThreads) + threadIdx.x;
                *cs++ = tk_comp(score_bits(b[u], ATTN), i - tl.seg0);
            }
    }
    def = block_sum(def, sm);
    if (threadIdx.x == 0) tile_def[blockIdx.x] = def;
}

// one radix-select step: the bin of h[0..256) holding the need-th largest (whole block calls;
// sh[0] = bin, sh[1] = need within it, sh[2] = its count)
__device__ __forceinline__ void tk_find_bin256(const uint32_t* h, uint32_t need, uint32_t* sh) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        uint32_t own = 0;
        for (int q = 0; q < 8; ++q) own += h[255 - 8 * lane - q];
        const uint32_t incl = warp_incl_scan(own);
        const uint32_t before = incl - own;
        if (own && before < need && before + own >= need) {
            uint32_t cum = before;
            for (int q = 0; q < 8; ++q) {
                const int bin = 255 - 8 * lane - q;
                if (cum + h[bin] >= need) {
                    sh[0] = (uint32_t)bin;
                    sh[1] = need - cum;
                    sh[2] = h[bin];
                    break;
                }
                cum += h[bin];
            }
        }
    }
    __syncthreads();
}

// need-th largest (1-based) of n distinct u64 keys at p (shared or global memory) that agree on
// every bit from `top` up (the candidates of one score bucket share its 11 top bits): digits of
// up to 8 bits from bit top - 1 down; stops as soon as one key is left with the prefix
__device__ uint64_t tk_select(const uint64_t* p, uint32_t n, uint32_t need, int top, uint32_t* h, uint32_t* sh,
                              uint64_t* shk) {
    const uint64_t fixed = top >= 64 ? 0ull : ~0ull << top;
    uint64_t prefix = n ? (p[0] & fixed) : 0ull, mask = fixed;
    for (int hi = top; hi > 0;) {
        const int wd = hi < 8 ? hi : 8, shf = hi - wd;
        hi = shf;
        for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            const uint64_t kk = p[i];
            if ((kk & mask) == prefix) atomicAdd(&h[(uint32_t)(kk >> shf) & ((1u << wd) - 1u)], 1u);
        }
        __syncthreads();
        tk_find_bin256(h, need, sh);
        prefix |= (uint64_t)sh[0] << shf;
        need = sh[1];
        mask |= (uint64_t)((1u << wd) - 1u) << shf;
        const bool single = sh[2] == 1u;
        __syncthreads();
        if (single) {
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
                if ((p[i] & mask) == prefix) *shk = p[i];
            __syncthreads();
            return *shk;
        }
    }
    return prefix;
}

// per segment: kstar (mode 2), the selected candidates per tile, then the exclusive output
// offsets of the segment's tiles
constexpr int kTkSelThreads = 512;
__global__ void __launch_bounds__(kTkSelThreads) topk_select_kernel(int bits, const uint32_t* __restrict__ seg_lo,
                                                                    const uint32_t* __restrict__ tile_start,
                                                                    const uint64_t* __restrict__ seg_off,
                                                                    TkSeg* __restrict__ seg,
                                                                    const uint64_t* __restrict__ cand,
                                                                    const uint32_t* __restrict__ cand_cnt,
                                                                    const uint32_t* __restrict__ tile_def,
                                                                    uint32_t* __restrict__ tile_sel,
                                                                    uint64_t* __restrict__ tile_off) {
    extern __shared__ __align__(16) uint64_t keys[];   // [kTkSmemCand]
    __shared__ uint32_t h[256];
    __shared__ uint32_t sh[4];
    __shared__ uint64_t shk;
    __shared__ uint64_t sm[33];
    const int64_t s = blockIdx.x;
    TkSeg st = seg[s];
    const uint32_t t0 = tile_start[s], t1 = tile_start[s + 1];
    const uint32_t seg0 = seg_lo[s];
    if (st.mode == 2u) {
        const uint32_t n = cand_cnt[s];
        const uint64_t* cs = cand + seg0;
        uint64_t kst;
        if (n <= kTkSmemCand) {
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) keys[i] = cs[i];
            __syncthreads();
            kst = tk_select(keys, n, st.need, 64 - bits, h, sh, &shk);   // (digit == b1: bits 64-bits.. fixed)
        } else {
            kst = tk_select(cs, n, st.need, 64 - bits, h, sh, &shk);   // (massive ties: the candidates stay in HBM)
        }
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            const uint64_t c = n <= kTkSmemCand ? keys[i] : cs[i];
            if (c >= kst) atomicAdd(&tile_sel[t0 + (0xffffffffu - (uint32_t)c) / (uint32_t)kTkTile], 1u);
        }
        if (threadIdx.x == 0) {
            st.kstar = kst;
            seg[s] = st;
        }
        __syncthreads();
    }
    uint64_t carry = seg_off[s];
    for (uint32_t base = t0; base < t1; base += blockDim.x) {
        const uint32_t t = base + threadIdx.x;
        uint64_t v = 0;
        if (t < t1) v = (uint64_t)tile_def[t] + (st.mode == 2u ? tile_sel[t] : 0u);
        uint64_t tot;
        const uint64_t ex = block_excl_scan(v, sm, &tot);
        if (t < t1) tile_off[t] = carry + ex;
        carry += tot;
        __syncthreads();
    }
}

// ordered compaction of one tile: 512 threads, warp w owns entries w*256 .. w*256+255 of the
// tile (8 groups of 32, coalesced), one ballot per group, warp totals scanned across the block
constexpr int kTkWThreads = 512;
constexpr int kTkWItems = kTkTile / kTkWThreads;   // 8
template <int ATTN>
__global__ void __launch_bounds__(kTkWThreads, 2) topk_write_kernel(Keys keys, const float* __restrict__ vals,
                                                                    const uint32_t* __restrict__ seg_lo,
                                                                    const uint32_t* __restrict__ tile_start,
                                                                    const uint32_t* __restrict__ tile_seg, int64_t nseg,
                                                                    int attn, int bits, const TkSeg* __restrict__ seg,
                                                                    const uint64_t* __restrict__ tile_off, KeysOut ok,
                                                                    float* __restrict__ ov, int64_t* __restrict__ osrc) {
    __shared__ uint32_t wc[kTkWThreads / 32];
    const TkTile tl = tk_tile(seg_lo, tile_start, tile_seg, nseg, blockIdx.x);
    if (!tl.ok) return;
    const TkSeg st = seg[tl.s];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t w0 = tl.lo + (uint32_t)warp * (32u * kTkWItems);
    const uint64_t pos0 = tile_off[blockIdx.x];
    uint32_t b[kTkWItems];
    uint64_t kk[kTkWItems];
#pragma unroll
    for (int u = 0; u < kTkWItems; ++u) {
        const uint32_t i = w0 + 32u * u + lane;
        b[u] = i < tl.hi ? __float_as_uint(__ldg(&vals[i])) : 0u;
        kk[u] = i < tl.hi ? keys[i] : 0ull;
    }
    unsigned m[kTkWItems];
    uint32_t c = 0;
#pragma unroll
    for (int u = 0; u < kTkWItems; ++u) {
        const uint32_t i = w0 + 32u * u + lane;
        const uint32_t sc = score_bits(b[u], ATTN);
        const uint32_t d = sc >> (32 - bits);
        const bool keep = i < tl.hi && (st.mode == 0u || d > st.b1 || (d == st.b1 && (st.mode == 1u ||
                                                                                     tk_comp(sc, i - tl.seg0) >= st.kstar)));
        m[u] = __ballot_sync(kFull, keep);
        c += (uint32_t)__popc(m[u]);
    }
    if (lane == 0) wc[warp] = c;
    __syncthreads();
    uint64_t pos = pos0;
    for (int q = 0; q < warp; ++q) pos += wc[q];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int u = 0; u < kTkWItems; ++u) {
        if ((m[u] >> lane) & 1u) {
            const uint32_t i = w0 + 32u * u + lane;
            const uint64_t o = pos + (uint32_t)__popc(m[u] & lt);
            ok.put(o, kk[u]);
            ov[o] = __uint_as_float(b[u]);
            if (osrc) osrc[o] = (int64_t)i;
        }
        pos += (uint32_t)__popc(m[u]);
    }
}

cudaError_t launch_topk(Keys keys, const float* vals, const uint32_t* seg_lo, int64_t nseg, int64_t nnz_bound,
                        int attn, int64_t k, const TopkBufs& w, KeysOut out_keys, float* out_vals,
                        int64_t* out_src, int64_t* out_nnz, cudaStream_t s) {
    if (nseg == 0) return cudaMemsetAsync(out_nnz, 0, sizeof(int64_t), s);
    const unsigned tiles = (unsigned)topk_tiles_bound(nnz_bound, nseg);
    const int bits = topk_bits(nnz_bound, nseg);
    cudaError_t e = cudaMemsetAsync(w.hist, 0, sizeof(uint32_t) * ((size_t)nseg << bits), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(w.tile_sel, 0, sizeof(uint32_t) * (size_t)tiles, s);
    if (e != cudaSuccess) return e;
    { SPC_PHASE("topk_plan", s, 1); topk_plan_kernel<<<1, 1024, 0, s>>>(seg_lo, nseg, k, w.seg_off, w.tile_start, out_nnz); }
    {
        SPC_PHASE("topk_plan", s, 1);
        topk_tile_map_kernel<<<(unsigned)std::min<int64_t>(nseg, 4096), 128, 0, s>>>(w.tile_start, nseg, w.tile_seg);
    }
    {
        SPC_PHASE("topk_hist", s, 1);
        (attn == SPC_ATTN_RAW ? topk_hist_kernel<SPC_ATTN_RAW> : topk_hist_kernel<SPC_ATTN_MAGNITUDE>)<<<(tiles + kTkHistTiles - 1) / kTkHistTiles, kTkThreads, 0, s>>>(vals, seg_lo, w.tile_start, w.tile_seg, nseg, attn, k, bits, w.hist);
    }
    { SPC_PHASE("topk_find", s, 1); topk_find_kernel<<<(unsigned)nseg, 256, 0, s>>>(seg_lo, k, bits, w.hist, w.seg, w.cand_cnt); }
    {
        SPC_PHASE("topk_collect", s, 1);
        (attn == SPC_ATTN_RAW ? topk_collect_kernel<SPC_ATTN_RAW> : topk_collect_kernel<SPC_ATTN_MAGNITUDE>)<<<tiles, kTkThreads, 0, s>>>(vals, seg_lo, w.tile_start, w.tile_seg, nseg, attn, bits, w.seg, w.cand,
                                                         w.cand_cnt, w.tile_def);
    }
    {
        SPC_PHASE("topk_select", s, 1);
        const size_t smem = kTkSmemCand * sizeof(uint64_t);
        cudaError_t ea = cudaFuncSetAttribute(topk_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (ea != cudaSuccess) return ea;
        topk_select_kernel<<<(unsigned)nseg, kTkSelThreads, smem, s>>>(bits, seg_lo, w.tile_start, w.seg_off, w.seg, w.cand,
                                                                   w.cand_cnt, w.tile_def, w.tile_sel, w.tile_off);
    }
    {
        SPC_PHASE("topk_write", s, 1);
        (attn == SPC_ATTN_RAW ? topk_write_kernel<SPC_ATTN_RAW> : topk_write_kernel<SPC_ATTN_MAGNITUDE>)<<<tiles, kTkWThreads, 0, s>>>(keys, vals, seg_lo, w.tile_start, w.tile_seg, nseg, attn, bits, w.seg,
                                                       w.tile_off, out_keys, out_vals, out_src);
    }
    return cudaGetLastError();
}

}  // namespace spc

// Streamed forward (variant S): the per-segment stages around the convolution passes of
// conv_fwd.cu. Alg. 1 keeps one dense buffer per (b, oc) and selects the k largest responses
// from it ("select k largest responses" P:80, Alabi et al. P:104). Here the dense
// responses never reach HBM:
//   sampled pass (conv_fwd_sample_kernel): score histograms of every sp_period-th tile;
//   find (this file):      per segment a threshold tlow whose estimated rank is a little above k;
//   main pass (conv_fwd_kernel): every support entry with score >= tlow ("candidates") is
//                          appended in key order to its tile's run;
//   resolve (this file):   the exact k-th largest composite key (score, ~p) among the candidates
//                          (reading R7: ties -> smaller key); a segment whose candidates cannot
//                          contain it (the sample missed) is queued for the redo pass, which
//                          recomputes its tiles with every support entry as a candidate;
//   tile scan + write:     ordered compaction of the kept candidates ("compress ids ...
//                          write").
// The result is exactly the selection of the dense-buffer algorithm: the candidates are a
// superset of the kept set whenever resolve accepts them.
#include "spc_internal.cuh"
#include "block_scan.cuh"

#include <cmath>

namespace spc {

__device__ __forceinline__ uint64_t comp_key(uint32_t sc, uint32_t p) {
    return ((uint64_t)sc << 32) | (uint64_t)(0xffffffffu - p);
}

// first voxel (within the segment) of tile t = x*nty + ty
__device__ __forceinline__ uint32_t tile_base(int t, int nty, int TY, int Y, int Z) {
    const int x = t / nty, ty = t - x * nty;
    return (uint32_t)(((int64_t)x * Y + (int64_t)ty * TY) * Z);
}

struct StreamGeo {
    int nty, TY, Y, Z;
    int64_t V;
};

// ------------------------------------------------------------------------------------ find
// tlow from the sampled histogram (bins = score >> 21). The sampled tiles are a fraction f of
// the segment; the threshold is placed where the sampled count above it reaches
// want = 1.08 k f + 4 sqrt(k f) + 8 (binomial margin of several sigma), interpolating inside the
// crossing bin. Segments whose estimated support is close to k (or whose sample is too small)
// take every support entry as a candidate (tlow = 0).
__global__ void stream_find_kernel(FwdArgs a, double f) {
    const int64_t s = blockIdx.x;
    __shared__ uint64_t sm[33];
    const uint32_t* h = a.hist + s * kSelBins;
    constexpr int per = kSelBins / 256;
    uint64_t local = 0;
    for (int q = 0; q < per; ++q) local += h[kSelBins - 1 - threadIdx.x * per - q];
    uint64_t tot;
    const uint64_t before = block_excl_scan(local, sm, &tot);
    const double k = (double)a.k;
    const double r = k * f;
    const double want = 1.08 * r + 4.0 * sqrt(r) + 8.0;
    const bool all = tot == 0 || (double)tot / f <= 1.1 * k + 64.0 || (double)tot < want;
    if (all) {
        if (threadIdx.x == 0) a.tlow[s] = 0u;
        return;
    }
    if ((double)before < want && (double)(before + local) >= want) {
        double cum = (double)before;
        for (int q = 0; q < per; ++q) {
            const int bin = kSelBins - 1 - threadIdx.x * per - q;
            const double hb = (double)h[bin];
            if (cum + hb >= want) {
                // large samples: interpolate inside the crossing bin; small ones (spatially
                // correlated surface data, discrete values with exact ties) take the bin's lower
                // edge, one bin lower below 2000 sampled entries -- a miss costs a redo pass
                uint32_t t;
                if ((double)tot >= 20000.0) {
                    const double frac = (want - cum) / hb;   // share of the bin needed, from its top
                    t = ((uint32_t)bin << 21) + (uint32_t)fmax(0.0, floor((1.0 - frac) * (double)(1u << 21)));
                } else {
                    const int b2 = (double)tot >= 2000.0 ? bin : max(0, bin - 1);
                    t = (uint32_t)b2 << 21;
                }
                a.tlow[s] = t;
                return;
            }
            cum += hb;
        }
    }
}

// --------------------------------------------------------------------------------- resolve
constexpr int kSRThreads = 512;
constexpr int kSRWarps = kSRThreads / 32;
constexpr int kSRCap = 4096;
#ifndef SPC_SR_GRANULE
#define SPC_SR_GRANULE 1
#endif   // candidates of the threshold bucket collected in shared memory

// Visit every candidate run of segment s: f.run(t, n) by one warp per tile run. Tiles are dealt
// to the warps in granules of G consecutive tiles (granule q -> warp q % kSRWarps); G = 1 spreads
// spatially clustered candidates (surfaces, strokes) over all warps (OctNet trunk resolve 1.28 ->
// 0.42 ms against G = 32; C4 is indifferent).
template <typename F>
__device__ __forceinline__ void for_candidates(const FwdArgs& a, int64_t s, F f) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t* tc = a.tcnt + s * a.ntile;
    constexpr int G = SPC_SR_GRANULE;
    auto tile_at = [&](int base, int j) { return base + (warp + kSRWarps * (j / G)) * G + (j % G); };
    for (int base = 0; base < a.ntile; base += kSRWarps * 32) {
        const int tl = tile_at(base, lane);
        const uint32_t mycnt = tl < a.ntile ? tc[tl] : 0u;
        unsigned any = __ballot_sync(kFull, mycnt != 0u);
        while (any) {
            const int j = __ffs(any) - 1;
            any &= any - 1;
            const uint32_t n = __shfl_sync(kFull, mycnt, j);
            f.run(tile_at(base, j), n);
        }
    }
}

// slot of the calling lane in a shared-memory list: one atomic per warp for the active lanes
__device__ __forceinline__ uint32_t warp_append(uint32_t* cnt) {
    const unsigned m = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(cnt, (uint32_t)__popc(m));
    base = __shfl_sync(m, base, leader);
    return base + (uint32_t)__popc(m & ((1u << lane) - 1u));
}

__device__ __forceinline__ uint32_t tile_of(uint32_t p, const StreamGeo& g) {
    const uint32_t yz = (uint32_t)g.Y * (uint32_t)g.Z;
    const uint32_t x = p / yz;
    const uint32_t y = (p - x * yz) / (uint32_t)g.Z;
    return x * (uint32_t)g.nty + y / (uint32_t)g.TY;
}

// The bin of histogram h[0..nb) holding the need-th largest entry (1 <= need <= total), found by
// warp 0 (the caller restricts it): 32 stripes of consecutive bins from the top, summed with a
// lane rotation (no bank conflicts), one warp scan, then the crossing lane walks its stripe.
// sh[0] = bin, sh[1] = need - (entries above the bin), sh[2] = h[bin].
__device__ __forceinline__ void warp_find_bin(const uint32_t* h, uint32_t nb, uint64_t need, uint64_t* sh) {
    const int lane = threadIdx.x & 31;
    const int per = (int)((nb + 31u) >> 5);
    uint32_t own = 0;
    for (int q = 0; q < per; ++q) {
        const int bin = (int)nb - 1 - per * lane - (q + lane) % per;
        if (bin >= 0) own += h[bin];
    }
    const uint32_t incl = warp_incl_scan(own);
    const uint64_t before = incl - own;
    const bool hit = own && before < need && before + own >= need;
    if (hit) {
        uint64_t cum = before;
        for (int q = 0; q < per; ++q) {
            const int bin = (int)nb - 1 - per * lane - q;
            if (bin < 0) break;
            if (cum + h[bin] >= need) {
                sh[0] = (uint64_t)bin;
                sh[1] = need - cum;
                sh[2] = h[bin];
                break;
            }
            cum += h[bin];
        }
    }
    const uint32_t total = __shfl_sync(kFull, incl, 31);
    if (!__any_sync(kFull, hit) && lane == 0) {   // unreachable for a valid need: bin 0
        const uint64_t above = total - h[0];
        sh[0] = 0;
        sh[1] = need > above ? need - above : 1;
        sh[2] = h[0];
    }
}

// need-th largest (1-based) of n distinct u64 keys in shared memory: radix select with 8-bit
// digits from the top (all threads of the block call it)
__device__ uint64_t smem_select(const uint64_t* keys, uint32_t n, uint32_t need, uint32_t* h256, uint64_t* sh) {
    uint64_t prefix = 0, mask = 0;
    for (int pass = 0; pass < 8; ++pass) {
        const int shf = 56 - 8 * pass;
        for (int i = threadIdx.x; i < 256; i += blockDim.x) h256[i] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            const uint64_t k = keys[i];
            if ((k & mask) == prefix) atomicAdd(&h256[(uint32_t)(k >> shf) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) warp_find_bin(h256, 256u, need, sh);
        __syncthreads();
        prefix |= sh[0] << shf;
        need = (uint32_t)sh[1];
        mask |= 255ull << shf;
        const bool single = sh[2] == 1u;   // one key left with this prefix: it is the answer
        __syncthreads();
        if (single) {
            for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
                if ((keys[i] & mask) == prefix) sh[3] = keys[i];
            __syncthreads();
            return sh[3];
        }
    }
    return prefix;
}

// the same select by one warp over its own key list (warp-per-segment resolve)
__device__ uint64_t warp_select(const uint64_t* keys, uint32_t n, uint32_t need, uint32_t* h256, uint64_t* sh) {
    const int lane = threadIdx.x & 31;
    uint64_t prefix = 0, mask = 0;
    for (int pass = 0; pass < 8; ++pass) {
        const int shf = 56 - 8 * pass;
        for (int i = lane; i < 256; i += 32) h256[i] = 0;
        __syncwarp();
        for (uint32_t i = lane; i < n; i += 32) {
            const uint64_t k = keys[i];
            if ((k & mask) == prefix) atomicAdd(&h256[(uint32_t)(k >> shf) & 255u], 1u);
        }
        __syncwarp();
        warp_find_bin(h256, 256u, need, sh);
        __syncwarp();
        prefix |= sh[0] << shf;
        need = (uint32_t)sh[1];
        mask |= 255ull << shf;
        const bool single = sh[2] == 1u;
        __syncwarp();
        if (single) {
            for (uint32_t i = lane; i < n; i += 32)
                if ((keys[i] & mask) == prefix) sh[3] = keys[i];
            __syncwarp();
            return sh[3];
        }
    }
    return prefix;
}

// pass 0: every segment; pass 1: only segments the redo pass recomputed
__global__ void __launch_bounds__(kSRThreads, 4) stream_resolve_kernel(FwdArgs a, StreamGeo g, int pass) {
    const int64_t s = blockIdx.x;
    if (pass == 1 && !a.fail[s]) return;
    const uint64_t n = a.cand_cur[s];
    const uint64_t k = (uint64_t)a.k;
    // With tlow = 0 every support entry is a candidate (n = |S|): keep all when |S| <= k. With
    // tlow > 0 the candidates hold the k largest iff there are at least k of them; otherwise the
    // segment is recomputed with tlow = 0 (whatever its support size).
    const bool tl0 = a.tlow[s] == 0u;
    const bool fail = !tl0 && (a.attn == SPC_ATTN_NONE || n < k);
    const bool keep_all = a.attn == SPC_ATTN_NONE || n <= k;   // (tlow = 0: n = |S|)
    if (fail) {
        if (pass == 0 && threadIdx.x == 0) {
            // the sampled threshold was too high: recompute this segment with tlow = 0
            a.fail[s] = 1;
            a.tlow[s] = 0;       // the redo pass keeps every support entry
            a.cand_cur[s] = 0;
            a.cmax[s] = 0;
            const int b = (int)(s / (int64_t)a.seg_stride);
            if (atomicExch(&a.bflag[b], 1) == 0) a.redo_b[atomicAdd(a.redo_n, 1)] = b;
        }
        return;   // (pass 1 cannot fail: with tlow = 0 the candidates are the whole support)
    }
    if (keep_all) {
        if (threadIdx.x == 0) {
            FwdSeg st{};
            st.keep_all = 1;
            a.seg[s] = st;
        }
        return;
    }
    __shared__ uint32_t h[kSelBins];
    __shared__ uint64_t keys[kSRCap];
    __shared__ uint64_t sh[4];
    __shared__ uint32_t sh_n;
    const uint32_t tl = a.tlow[s];
    const uint32_t mxr = a.cmax[s] - tl;
    const int sh1 = max(0, 32 - __clz(mxr) - 11);   // (score - tl) >> sh1 < 2048
    const int attn = a.attn;
    const float* cval = a.cval + s * g.V;
    const uint32_t* cpos = a.cpos + s * g.V;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) sh_n = 0;
    __syncthreads();
    if (n <= (uint64_t)kSRCap) {
        // small candidate sets (MNIST-like layers, small grids): every candidate's composite key
        // in shared memory in one pass, the k-th largest by ranking (n <= 256) or radix select
        struct AllF {
            const float* cv; const uint32_t* cp; uint64_t* keys; uint32_t* sh_n; uint32_t* tdef; int attn, lane;
            const StreamGeo* g;
            __device__ void run(int t, uint32_t n) const {
                const uint32_t b0 = tile_base(t, g->nty, g->TY, g->Y, g->Z);
                for (uint32_t i = lane; i < n; i += 32)
                    {
                    const uint64_t key = comp_key(score_bits(__float_as_uint(cv[b0 + i]), attn), cp[b0 + i]);
                    keys[warp_append(sh_n)] = key;
                }
                if (lane == 0) tdef[t] = 0;
            }
        } af{cval, cpos, keys, &sh_n, a.tile_def + s * a.ntile, attn, lane, &g};
        for_candidates(a, s, af);
        __syncthreads();
        const uint32_t ns = sh_n;
        uint64_t kst;
        if (ns <= 256u) {
            if (threadIdx.x == 0) sh[0] = 0;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) {   // rank = keys above (all distinct)
                const uint64_t ki = keys[i];
                uint32_t above = 0;
                for (uint32_t j = 0; j < ns; ++j) above += keys[j] > ki ? 1u : 0u;
                if (above == (uint32_t)k - 1u) sh[0] = ki;
            }
            __syncthreads();
            kst = sh[0];
        } else {
            kst = smem_select(keys, ns, (uint32_t)k, h, sh);
        }
        uint32_t* tsel = a.tile_sel + s * a.ntile;
        for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x)
            if (keys[i] >= kst) atomicAdd(&tsel[tile_of(0xffffffffu - (uint32_t)keys[i], g)], 1u);
        if (threadIdx.x == 0) {
            FwdSeg st{};
            st.keep_all = 0;
            st.kstar = kst;
            a.seg[s] = st;
        }
        return;
    }
    // ---- histogram of the candidates' score digit (precomputed by stream_resolve_hist_kernel when
    // the segments are fewer than the SMs)
    if (a.rhist) {
        for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) h[i] = a.rhist[s * kSelBins + i];
    } else {
    for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    struct HistF {
        const float* cv; uint32_t* h; uint32_t tl; int sh1, attn, lane; const StreamGeo* g;
        __device__ void run(int t, uint32_t n) const {
            const float* v = cv + tile_base(t, g->nty, g->TY, g->Y, g->Z);
            for (uint32_t i0 = lane; i0 < n; i0 += 128) {   // four loads in flight per lane
                uint32_t vb[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) vb[q] = i0 + 32u * q < n ? __float_as_uint(v[i0 + 32u * q]) : 0u;
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (i0 + 32u * q < n) atomicAdd(&h[(score_bits(vb[q], attn) - tl) >> sh1], 1u);
            }
        }
    } hf{cval, h, tl, sh1, attn, lane, &g};
    for_candidates(a, s, hf);
    }
    __syncthreads();
    // ---- bucket of the k-th from the top
    if (threadIdx.x < 32) {
        constexpr int per = kSelBins / 32;
        uint32_t own = 0;
        for (int q = 0; q < per; ++q) own += h[kSelBins - 1 - per * lane - q];
        const uint32_t incl = warp_incl_scan(own);
        const uint64_t before = incl - own;
        if (own && before < k && before + own >= k) {
            uint64_t cum = before;
            for (int q = 0; q < per; ++q) {
                const int bin = kSelBins - 1 - per * lane - q;
                if (cum + h[bin] >= k) {
                    sh[0] = (uint64_t)bin;
                    sh[1] = k - cum;       // need within the bucket
                    sh[2] = h[bin];
                    break;
                }
                cum += h[bin];
            }
        }
    }
    __syncthreads();
    const uint32_t B = (uint32_t)sh[0];
    uint64_t need = sh[1];
    uint64_t bcnt = sh[2];
    // Within the bucket, the order is that of K' = ((score - lo) << 32) | ~p (lo = the bucket's
    // lowest score): a key of W = sh1 + 32 bits. Narrow it with 11-bit digits over the HBM list
    // until the survivors fit shared memory (usually no narrowing at all).
    const uint32_t lo = tl + (B << sh1);
    uint64_t pre = 0;   // survivors: (K' >> pos) == pre
    int pos = sh1 + 32;
    auto kprime = [&](uint32_t sc, uint32_t p) -> uint64_t {
        return ((uint64_t)(sc - lo) << 32) | (uint64_t)(0xffffffffu - p);
    };
    while (bcnt > (uint64_t)kSRCap) {
        const int d = min(11, pos);
        pos -= d;
        const uint32_t nb = 1u << d;
        for (uint32_t i = threadIdx.x; i < nb; i += blockDim.x) h[i] = 0;
        __syncthreads();
        struct NarrowF {
            const float* cv; const uint32_t* cp; uint32_t* h; uint32_t tl, lo; uint32_t B; int sh1, attn, lane, pos, d;
            uint64_t pre; const StreamGeo* g;
            __device__ void run(int t, uint32_t n) const {
                const uint32_t b0 = tile_base(t, g->nty, g->TY, g->Y, g->Z);
                for (uint32_t i = lane; i < n; i += 32) {
                    const uint32_t sc = score_bits(__float_as_uint(cv[b0 + i]), attn);
                    if (((sc - tl) >> sh1) != B) continue;
                    const uint64_t kp = ((uint64_t)(sc - lo) << 32) | (uint64_t)(0xffffffffu - cp[b0 + i]);
                    if ((kp >> (pos + d)) == pre) atomicAdd(&h[(uint32_t)(kp >> pos) & ((1u << d) - 1u)], 1u);
                }
            }
        } nf{cval, cpos, h, tl, lo, B, sh1, attn, lane, pos, d, pre, &g};
        for_candidates(a, s, nf);
        __syncthreads();
        if (threadIdx.x < 32) warp_find_bin(h, nb, need, sh);
        __syncthreads();
        pre = (pre << d) | sh[0];
        need = sh[1];
        bcnt = sh[2];
        __syncthreads();
    }
    if (a.rhist) {   // split resolve: the collect runs on several CTAs per segment, then the select
        if (threadIdx.x == 0) {
            ResolveState r{};
            r.pre = pre;
            r.need = need;
            r.B = B;
            r.lo = lo;
            r.pos = pos;
            r.sh1 = sh1;
            r.active = 1;
            a.rstate[s] = r;
        }
        return;
    }
    // ---- collect the survivors; per tile run count the entries ranked above them ("definite")
    struct CollectF {
        const float* cv; const uint32_t* cp; uint64_t* keys; uint32_t* sh_n; uint32_t* tdef;
        uint32_t tl, lo, B; int sh1, attn, lane, pos; uint64_t pre; const StreamGeo* g;
        __device__ void run(int t, uint32_t n) const {
            const uint32_t b0 = tile_base(t, g->nty, g->TY, g->Y, g->Z);
            uint32_t def = 0;
            for (uint32_t i0 = lane; i0 < n; i0 += 128) {   // four loads in flight per lane
                uint32_t vb[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) vb[q] = i0 + 32u * q < n ? __float_as_uint(cv[b0 + i0 + 32u * q]) : 0u;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t i = i0 + 32u * q;
                    if (i >= n) continue;
                    const uint32_t sc = score_bits(vb[q], attn);
                    const uint32_t dg = (sc - tl) >> sh1;
                    if (dg > B) { ++def; continue; }
                    if (dg < B) continue;
                    const uint32_t p = cp[b0 + i];
                    const uint64_t kp = ((uint64_t)(sc - lo) << 32) | (uint64_t)(0xffffffffu - p);
                    const uint64_t top = kp >> pos;
                    if (top > pre) ++def;
                    else if (top == pre) keys[atomicAdd(sh_n, 1u)] = kp;
                }
            }
            def = warp_sum(def);
            if (lane == 0) tdef[t] = def;
        }
    } cf{cval, cpos, keys, &sh_n, a.tile_def + s * a.ntile, tl, lo, B, sh1, attn, lane, pos, pre, &g};
    // (tile_def is written for every run with candidates; the tile scan reads no other)
    for_candidates(a, s, cf);
    __syncthreads();
    const uint32_t ns = sh_n;
    const uint64_t kps = smem_select(keys, ns, (uint32_t)need, h, sh);
    // kept iff K' >= kps among the survivors; per tile run the selected survivors
    uint32_t* tsel = a.tile_sel + s * a.ntile;
    for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) {
        const uint64_t kp = keys[i];
        if (kp >= kps) atomicAdd(&tsel[tile_of(0xffffffffu - (uint32_t)kp, g)], 1u);
    }
    if (threadIdx.x == 0) {
        FwdSeg st{};
        st.keep_all = 0;
        st.kstar = ((uint64_t)(lo + (uint32_t)(kps >> 32)) << 32) | (kps & 0xffffffffull);
        a.seg[s] = st;
    }
}

// Segments of at most kSmallV voxels (MNIST-like layers, coarse grids): one warp per segment, no
// block barriers. Every candidate's composite key goes to the warp's shared list (n <= V), the
// k-th largest by warp_select; same outcome and outputs as stream_resolve_kernel.
constexpr int kSmallV = 1024;
constexpr int kSmallWarps = 4;

__global__ void __launch_bounds__(32 * kSmallWarps) stream_resolve_small_kernel(FwdArgs a, StreamGeo g, int pass) {
    __shared__ uint64_t keys_all[kSmallWarps][kSmallV];
    __shared__ uint32_t h_all[kSmallWarps][256];
    __shared__ uint64_t sh_all[kSmallWarps][4];
    __shared__ uint32_t n_all[kSmallWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t s = (int64_t)blockIdx.x * kSmallWarps + warp;
    if (s >= a.nseg) return;                       // (warp-uniform, as every return below)
    if (pass == 1 && !a.fail[s]) return;
    const uint64_t n = a.cand_cur[s];
    const uint64_t k = (uint64_t)a.k;
    // With tlow = 0 every support entry is a candidate (n = |S|): keep all when |S| <= k. With
    // tlow > 0 the candidates hold the k largest iff there are at least k of them; otherwise the
    // segment is recomputed with tlow = 0 (whatever its support size).
    const bool tl0 = a.tlow[s] == 0u;
    const bool fail = !tl0 && (a.attn == SPC_ATTN_NONE || n < k);
    const bool keep_all = a.attn == SPC_ATTN_NONE || n <= k;   // (tlow = 0: n = |S|)
    if (fail) {
        if (pass == 0 && lane == 0) {
            a.fail[s] = 1;
            a.tlow[s] = 0;
            a.cand_cur[s] = 0;
            a.cmax[s] = 0;
            const int b = (int)(s / (int64_t)a.seg_stride);
            if (atomicExch(&a.bflag[b], 1) == 0) a.redo_b[atomicAdd(a.redo_n, 1)] = b;
        }
        return;
    }
    if (keep_all) {
        if (lane == 0) {
            FwdSeg st{};
            st.keep_all = 1;
            a.seg[s] = st;
        }
        return;
    }
    uint64_t* keys = keys_all[warp];
    uint32_t* cnt = &n_all[warp];
    if (lane == 0) *cnt = 0;
    __syncwarp();
    const float* cv = a.cval + s * g.V;
    const uint32_t* cp = a.cpos + s * g.V;
    const uint32_t* tc = a.tcnt + s * a.ntile;
    uint32_t* tdef = a.tile_def + s * a.ntile;
    const int attn = a.attn;
    for (int t0 = 0; t0 < a.ntile; t0 += 32) {
        const uint32_t mycnt = t0 + lane < a.ntile ? tc[t0 + lane] : 0u;
        unsigned any = __ballot_sync(kFull, mycnt != 0u);
        while (any) {
            const int j = __ffs(any) - 1;
            any &= any - 1;
            const int t = t0 + j;
            const uint32_t rn = __shfl_sync(kFull, mycnt, j);
            const uint32_t b0 = tile_base(t, g.nty, g.TY, g.Y, g.Z);
            for (uint32_t i = lane; i < rn; i += 32) {
                const uint64_t key = comp_key(score_bits(__float_as_uint(cv[b0 + i]), attn), cp[b0 + i]);
                const uint32_t slot = warp_append(cnt);
                if (slot < (uint32_t)kSmallV) keys[slot] = key;
            }
            if (lane == 0) tdef[t] = 0;   // every kept entry is counted in tile_sel
        }
    }
    __syncwarp();
    const uint32_t ns = min(*cnt, (uint32_t)kSmallV);
    const uint64_t kst = warp_select(keys, ns, (uint32_t)k, h_all[warp], sh_all[warp]);
    uint32_t* tsel = a.tile_sel + s * a.ntile;
    for (uint32_t i = lane; i < ns; i += 32)
        if (keys[i] >= kst) atomicAdd(&tsel[tile_of(0xffffffffu - (uint32_t)keys[i], g)], 1u);
    if (lane == 0) {
        FwdSeg st{};
        st.keep_all = 0;
        st.kstar = kst;
        a.seg[s] = st;
    }
}

// ------------------------------------------------------------------------- tile scan / write
// per segment: kept entries per tile run -> exclusive offsets; segment total -> kept[s]
__global__ void stream_tile_scan_kernel(FwdArgs a, uint64_t* kept) {
    const int64_t s = blockIdx.x;
    __shared__ uint64_t sm[33];
    const bool all = a.seg[s].keep_all != 0;
    uint64_t carry = 0;
    for (int64_t base = 0; base < a.ntile; base += blockDim.x) {
        const int64_t t = base + threadIdx.x;
        uint64_t v = 0;
        if (t < a.ntile) {
            const int64_t it = s * a.ntile + t;
            const uint32_t c = a.tcnt[it];
            v = (all || c == 0) ? (uint64_t)c : (uint64_t)a.tile_def[it] + a.tile_sel[it];
        }
        uint64_t tot;
        const uint64_t ex = block_excl_scan(v, sm, &tot);
        if (t < a.ntile) a.tile_off[s * a.ntile + t] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) kept[s] = carry;
}

// one warp per tile run: keep iff composite(score, p) >= kstar (every candidate when keep-all),
// ordered compaction ("compress ids from kD to 1D, write as sparse output")
constexpr int kSWWarps = 8;
template <bool K32>
__global__ void __launch_bounds__(32 * kSWWarps) stream_write_kernel(FwdArgs a, StreamGeo g) {
    const int lane = threadIdx.x & 31;
    const int64_t it = (int64_t)blockIdx.x * kSWWarps + (threadIdx.x >> 5);
    if (it >= a.nseg * a.ntile) return;
    const uint32_t n = a.tcnt[it];
    if (n == 0) return;
    const int64_t s = it / a.ntile;
    const int t = (int)(it - s * a.ntile);
    const FwdSeg st = a.seg[s];
    const uint32_t b0 = tile_base(t, g.nty, g.TY, g.Y, g.Z);
    const uint32_t* ip = a.cpos + s * g.V + b0;
    const float* iv = a.cval + s * g.V + b0;
    uint64_t out = a.seg_off[s] + a.tile_off[it];
    const uint64_t kb = ((uint64_t)a.seg0 + (uint64_t)s) * (uint64_t)g.V;
    const uint32_t ks = (uint32_t)(st.kstar >> 32), kp = (uint32_t)st.kstar;
    for (uint32_t i0 = 0; i0 < n; i0 += 128) {   // four groups of 32 loaded before any is used
        uint32_t pp[4], vb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t i = i0 + 32u * q + lane;
            pp[q] = i < n ? ip[i] : 0u;
            vb[q] = i < n ? __float_as_uint(iv[i]) : 0u;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const bool ok = i0 + 32u * q + lane < n;
            const uint32_t sc = score_bits(vb[q], a.attn);
            const bool keep = ok && (st.keep_all || sc > ks || (sc == ks && 0xffffffffu - pp[q] >= kp));
            const unsigned m = __ballot_sync(kFull, keep);
            if (keep) {
                const uint64_t o = out + __popc(m & ((1u << lane) - 1u));
                a.out_keys.template put_t<K32>(o, kb + pp[q]);
                a.out_vals[o] = __uint_as_float(vb[q]);
            }
            out += __popc(m);
        }
    }
}

// The resolve's candidate histogram with gridDim.y CTAs per segment (segments fewer than SMs):
// the same early outs and digit as stream_resolve_kernel; CTA part takes tiles part, part + P, ...
// (one warp per tile run), shared bins flushed to a.rhist with atomics.
__global__ void __launch_bounds__(256) stream_resolve_hist_kernel(FwdArgs a, StreamGeo g, int pass) {
    const int64_t s = blockIdx.x;
    if (pass == 1 && !a.fail[s]) return;
    const uint64_t n = a.cand_cur[s];
    const uint64_t k = (uint64_t)a.k;
    const bool tl0 = a.tlow[s] == 0u;
    const bool fail = !tl0 && (a.attn == SPC_ATTN_NONE || n < k);
    const bool keep_all = a.attn == SPC_ATTN_NONE || n <= k;
    if (fail || keep_all || n <= (uint64_t)kSRCap) return;
    __shared__ uint32_t h[kSelBins];
    for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint32_t tl = a.tlow[s];
    const uint32_t mxr = a.cmax[s] - tl;
    const int sh1 = max(0, 32 - __clz(mxr) - 11);
    const int attn = a.attn;
    const float* cval = a.cval + s * g.V;
    const uint32_t* tc = a.tcnt + s * a.ntile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int P = gridDim.y;
    for (int t = blockIdx.y + P * warp; t < a.ntile; t += P * nw) {
        const uint32_t cnt = tc[t];
        if (!cnt) continue;
        const float* v = cval + tile_base(t, g.nty, g.TY, g.Y, g.Z);
        for (uint32_t i0 = lane; i0 < cnt; i0 += 128) {
            uint32_t vb[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) vb[q] = i0 + 32u * q < cnt ? __float_as_uint(v[i0 + 32u * q]) : 0u;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (i0 + 32u * q < cnt) atomicAdd(&h[(score_bits(vb[q], attn) - tl) >> sh1], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kSelBins; i += blockDim.x)
        if (h[i]) atomicAdd(&a.rhist[s * kSelBins + i], h[i]);
}

// Split resolve, collect: the survivors of the threshold bucket (K' >> pos == pre) appended to the
// segment's global list, and per tile run the entries ranked above them (tile_def); CTA part
// takes tiles part, part + P, ... (one warp per tile run), as stream_resolve_kernel's CollectF.
__global__ void __launch_bounds__(256) stream_resolve_collect_kernel(FwdArgs a, StreamGeo g) {
    const int64_t s = blockIdx.x;
    const ResolveState r = a.rstate[s];
    if (!r.active) return;
    const uint32_t tl = a.tlow[s];
    const int attn = a.attn;
    const float* cv = a.cval + s * g.V;
    const uint32_t* cp = a.cpos + s * g.V;
    const uint32_t* tc = a.tcnt + s * a.ntile;
    uint32_t* tdef = a.tile_def + s * a.ntile;
    uint64_t* surv = a.rsurv + s * (int64_t)kSRCap;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int P = gridDim.y;
    for (int t = blockIdx.y + P * warp; t < a.ntile; t += P * nw) {
        const uint32_t n = tc[t];
        if (!n) continue;
        const uint32_t b0 = tile_base(t, g.nty, g.TY, g.Y, g.Z);
        uint32_t def = 0;
        for (uint32_t i0 = 0; i0 < n; i0 += 32) {
            const uint32_t i = i0 + lane;
            bool put = false;
            uint64_t kp = 0;
            if (i < n) {
                const uint32_t sc = score_bits(__float_as_uint(cv[b0 + i]), attn);
                const uint32_t dg = (sc - tl) >> r.sh1;
                if (dg > r.B) {
                    ++def;
                } else if (dg == r.B) {
                    kp = ((uint64_t)(sc - r.lo) << 32) | (uint64_t)(0xffffffffu - cp[b0 + i]);
                    const uint64_t top = kp >> r.pos;
                    if (top > r.pre) ++def;
                    else put = top == r.pre;
                }
            }
            const unsigned m = __ballot_sync(kFull, put);
            if (m) {
                uint32_t base = 0;
                if (lane == __ffs(m) - 1) base = atomicAdd(&a.rsurv_n[s], (uint32_t)__popc(m));
                base = __shfl_sync(kFull, base, __ffs(m) - 1);
                if (put) {
                    const uint32_t o = base + __popc(m & ((1u << lane) - 1u));
                    if (o < (uint32_t)kSRCap) surv[o] = kp;
                }
            }
        }
        def = warp_sum(def);
        if (lane == 0) tdef[t] = def;
    }
}

// Split resolve, select: the k-th of the survivors (smem_select), per tile run the selected ones.
__global__ void __launch_bounds__(kSRThreads) stream_resolve_select_kernel(FwdArgs a, StreamGeo g) {
    const int64_t s = blockIdx.x;
    const ResolveState r = a.rstate[s];
    if (!r.active) return;
    __shared__ uint32_t h[kSelBins];
    __shared__ uint64_t keys[kSRCap];
    __shared__ uint64_t sh[4];
    const uint32_t ns = min(a.rsurv_n[s], (uint32_t)kSRCap);
    for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) keys[i] = a.rsurv[s * (int64_t)kSRCap + i];
    __syncthreads();
    const uint64_t kps = smem_select(keys, ns, (uint32_t)r.need, h, sh);
    uint32_t* tsel = a.tile_sel + s * a.ntile;
    for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) {
        const uint64_t kp = keys[i];
        if (kp >= kps) atomicAdd(&tsel[tile_of(0xffffffffu - (uint32_t)kp, g)], 1u);
    }
    if (threadIdx.x == 0) {
        FwdSeg st{};
        st.keep_all = 0;
        st.kstar = ((uint64_t)(r.lo + (uint32_t)(kps >> 32)) << 32) | (kps & 0xffffffffull);
        a.seg[s] = st;
    }
}

cudaError_t launch_stream_find(const FwdArgs& a, cudaStream_t s) {
    const double f = (double)a.nsamp / (double)a.ntile;
    SPC_PHASE("fwd_find", s, 1);
    stream_find_kernel<<<(unsigned)a.nseg, 256, 0, s>>>(a, f);
    return cudaGetLastError();
}

cudaError_t launch_stream_resolve(const Geo& gy, const FwdTile& t, const FwdArgs& a, int pass, cudaStream_t s) {
    const StreamGeo g{t.nty, t.TY, gy.Y, gy.Z, gy.V};
    const bool split = a.rhist && gy.V > kSmallV;
    SPC_PHASE(pass == 0 ? "fwd_resolve" : "fwd_resolve_redo", s, split ? 4 : 1);
    const int parts = (int)std::max<int64_t>(2, std::min<int64_t>(64, (int64_t)num_sms() * 4 / std::max<int64_t>(a.nseg, 1)));
    if (split) {
        cudaError_t e = cudaMemsetAsync(a.rhist, 0, (size_t)a.nseg * kSelBins * sizeof(uint32_t), s);
        if (e == cudaSuccess) e = cudaMemsetAsync(a.rstate, 0, (size_t)a.nseg * sizeof(ResolveState), s);
        if (e == cudaSuccess) e = cudaMemsetAsync(a.rsurv_n, 0, (size_t)a.nseg * sizeof(uint32_t), s);
        if (e != cudaSuccess) return e;
        stream_resolve_hist_kernel<<<dim3((unsigned)a.nseg, (unsigned)parts), 256, 0, s>>>(a, g, pass);
        stream_resolve_kernel<<<(unsigned)a.nseg, kSRThreads, 0, s>>>(a, g, pass);
        stream_resolve_collect_kernel<<<dim3((unsigned)a.nseg, (unsigned)parts), 256, 0, s>>>(a, g);
        stream_resolve_select_kernel<<<(unsigned)a.nseg, kSRThreads, 0, s>>>(a, g);
        return cudaGetLastError();
    }
    if (gy.V <= kSmallV)
        stream_resolve_small_kernel<<<(unsigned)((a.nseg + kSmallWarps - 1) / kSmallWarps), 32 * kSmallWarps, 0, s>>>(a, g, pass);
    else
        stream_resolve_kernel<<<(unsigned)a.nseg, kSRThreads, 0, s>>>(a, g, pass);
    return cudaGetLastError();
}

cudaError_t launch_stream_tail(const Geo& gy, const FwdTile& t, const FwdArgs& a, cudaStream_t s) {
    const StreamGeo g{t.nty, t.TY, gy.Y, gy.Z, gy.V};
    { SPC_PHASE("fwd_tile_scan", s, 1); stream_tile_scan_kernel<<<(unsigned)a.nseg, 256, 0, s>>>(a, a.cand_cnt); }
    cudaError_t e = launch_seg_scan_u64(a.cand_cnt, a.seg_off, a.nseg, a.out_nnz, a.out_append, s);
    if (e != cudaSuccess) return e;
    const int64_t runs = a.nseg * a.ntile;
    SPC_PHASE("fwd_write", s, 1);
    const unsigned grid = (unsigned)((runs + kSWWarps - 1) / kSWWarps);
    if (a.out_keys.k32) stream_write_kernel<true><<<grid, 32 * kSWWarps, 0, s>>>(a, g);
    else stream_write_kernel<false><<<grid, 32 * kSWWarps, 0, s>>>(a, g);
    return cudaGetLastError();
}

}  // namespace spc

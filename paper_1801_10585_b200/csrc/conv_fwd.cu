// Forward direct sparse convolution with attention, Alg. 1:
//   "for ic / for {id,val} in data(b,ic) / for {fid,fval} in filter(oc,ic): add val*fval to
//    buffer at uid", "get non-zero entries", "add bias",
//   "select k largest responses", "compress ids and write".
//
// B200 mapping. The paper keeps one dense buffer per (b, oc)
// in global memory and updates it with fp32 atomics one (b, oc) at a time.
// Here a CTA owns a tile = one x-plane, rows [y0, y0+TY) of full z-rows, for a group of ocg
// output channels; its slice of the buffer lives in shared memory and all tiles run at once.
// Warp w owns TY/8 consecutive output rows. For every (ic, in-plane offset (dx,dy)) the warp
// reads the contiguous run of stored inputs whose targets fall in its rows; lanes take 32
// inputs, the warp walks the weights of (ic, dx, dy, oc-group): all lanes share one weight, so
// the 32 read-modify-writes of a step hit 32 distinct voxels and no other warp writes them.
// No atomics, and a fixed loop order makes every recomputation bit-identical, which the
// attention pipeline relies on:
//   pass 1 (HIST):     support size and an 11-bit score-digit histogram per (b, oc);
//   find:              threshold digit B1 and `need` per (b, oc) (or keep-all);
//   pass 2 (CLASSIFY): entries with digit > B1 are kept (counted per tile), digit == B1 go
//                      to a candidate list;
//   resolve:           exact selection of `need` candidates by the composite key
//                      (score, ~p) -> kstar (reading R7: ties -> smaller key);
//   pass 3 (WRITE):    keep composite >= kstar, ordered compaction per tile at offsets
//                      scanned from the per-tile counts.
// The structural support (reading R3) is the set of voxels touched by any update: words start
// as an absent marker (a NaN pattern) that the first update replaces.
#include "spc_internal.cuh"
#include "block_scan.cuh"

#include <algorithm>
#ifdef SPC_DEBUG
#include <cstdio>
#endif

namespace spc {

constexpr int kFwdThreads = 256;
constexpr int kFwdWarps = kFwdThreads / 32;
constexpr size_t kFwdBudget = 108 * 1024;   // two CTAs (16 warps) per SM
constexpr int kStageCap = 2048;             // staged input entries per chunk of input channels
static_assert(2 * kStageCap >= kSelBins, "the epilogue histogram reuses the stage buffer");

// shared-memory bytes beyond the accumulator
static size_t fwd_fixed_smem(const KGeo& kg, int c_in, int TY, int64_t nwg) {
    auto r4 = [](size_t n) { return (n + 3) & ~(size_t)3; };
    const size_t PK = (size_t)c_in * kg.kx, G = (size_t)c_in * kg.kx * kg.ky;
    return 4 * (256 + 4 * r4((size_t)nwg) + r4(G + 1) + r4(PK * (TY + 2 * kg.hy + 1)) + r4(PK + 1) +
                2 * (size_t)kStageCap) + 64;
}

FwdTile plan_fwd_tile(const Geo& gy, const KGeo& kg, int c_out, int c_in, int64_t nw_total) {
    FwdTile t{};
    const int ZR = ((gy.Z + 2 * kg.hz + 3) / 4) * 4;
    const int pad = ((kg.hz + 3) / 4) * 4;
    const size_t row_b = (size_t)ZR * sizeof(float);
    auto need = [&](int ocg, int TY) {
        const int64_t nwg = std::min<int64_t>(nw_total, (int64_t)ocg * c_in * kg.KV);
        return fwd_fixed_smem(kg, c_in, TY, nwg) + (size_t)ocg * TY * row_b + (size_t)pad * 8;
    };
    // prefer >= 8 rows per warp (lane utilisation), then the largest group of channels
    int TY = std::min(gy.Y, 8 * kFwdWarps);
    int ocg = std::min(c_out, 16);
    while (ocg > 1 && need(ocg, TY) > kFwdBudget) --ocg;
    while (TY > 1 && need(ocg, TY) > kFwdBudget) --TY;          // ocg == 1: shorter tiles
    if (need(ocg, TY) > kFwdBudget) { t.smem = 0; return t; }
    while (TY < gy.Y && need(ocg, TY + kFwdWarps) <= kFwdBudget) TY += kFwdWarps;   // spare room
    TY = std::min(TY, std::min(gy.Y, 240));   // staged rows are packed in 8 bits (TY + 2*hy < 256)
    t.TY = TY;
    t.RW = (TY + kFwdWarps - 1) / kFwdWarps;
    t.nty = (gy.Y + TY - 1) / TY;
    t.ocg = ocg;
    t.n_ocg = (c_out + ocg - 1) / ocg;
    t.ZR = ZR;
    t.pad = pad;
    t.NT = gy.X * t.nty;
    t.nwg_max = (int)std::min<int64_t>(nw_total, (int64_t)ocg * c_in * kg.KV);
    t.smem = need(ocg, TY);
    return t;
}

// fast y = L / Z for L < 2^24 (float reciprocal + one correction each way)
__device__ __forceinline__ uint32_t div_small(uint32_t L, uint32_t Z, float invZ) {
    uint32_t q = __float2uint_rz(__uint2float_rz(L) * invZ);
    if (q * Z > L) --q;
    if ((q + 1) * Z <= L) ++q;
    return q;
}

__device__ __forceinline__ uint64_t composite(uint32_t sc, uint32_t p) {
    return ((uint64_t)sc << 32) | (uint64_t)(0xffffffffu - p);
}

__global__ void __launch_bounds__(kFwdThreads, 2)
conv_fwd_kernel(Geo gx, Geo gy, KGeo kg, FwdTile t, FwdArgs a) {
    extern __shared__ __align__(16) float smf[];
    const int c_in = (int)gx.C, c_out = (int)gy.C;
    const int Z = gy.Z, ZR = t.ZR;
    const int64_t tile = blockIdx.x;                 // (b, x, ty) flattened
    const int ty = (int)(tile % t.nty);
    const int x = (int)((tile / t.nty) % gy.X);
    const int64_t b = tile / ((int64_t)t.nty * gy.X);
    const int oc0 = blockIdx.y * t.ocg;
    const int nocl = min(t.ocg, c_out - oc0);
    const int y0 = ty * t.TY, ye = min(y0 + t.TY, gy.Y);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int TYZR = t.TY * ZR;

    // shared layout (float offsets, 16-byte aligned pieces):
    // [pad][acc ocg*TY*ZR][pad] | misc(256) | sw4 | swoff | rp | sbase | stage (= hist in the epilogue)
    const int KXY = kg.kx * kg.ky;
    const int G = c_in * KXY;                        // (ic, dx, dy) weight groups
    const int PK = c_in * kg.kx;                     // (ic, input plane) work items
    const int ylo = max(0, y0 - kg.hy), yhi = min(gy.Y, ye + kg.hy);
    const int nr = yhi - ylo;                        // input rows read per plane
    const int NRP = nr + 1;
    const int nw4 = (t.nwg_max + 3) & ~3;
    float* acc = smf + t.pad;
    uint32_t* misc = reinterpret_cast<uint32_t*>(smf + 2 * t.pad + t.ocg * TYZR);
    // per weight {acc offset of its target, value bits, row offset oy, 0}
    int4* sw4 = reinterpret_cast<int4*>(misc + 256);
    int* swoff = reinterpret_cast<int*>(sw4 + nw4);   // [G + 1] first weight of each (ic, dx, dy)
    uint32_t* rp = reinterpret_cast<uint32_t*>(swoff + ((G + 1 + 3) & ~3));
    int* sbase = reinterpret_cast<int*>(rp + ((PK * (t.TY + 2 * kg.hy + 1) + 3) & ~3));
    uint2* stage = reinterpret_cast<uint2*>(sbase + ((PK + 1 + 3) & ~3));
    uint32_t* hist = reinterpret_cast<uint32_t*>(stage);   // epilogue only

    {
        const int n4 = (2 * t.pad + t.ocg * TYZR) / 4;
        uint4 ab = make_uint4(kAbsent, kAbsent, kAbsent, kAbsent);
        for (int i = threadIdx.x; i < n4; i += blockDim.x) reinterpret_cast<uint4*>(smf)[i] = ab;
    }
    // this group's weights, ordered by (ic, dx, dy): "filter(oc, ic)" of Alg. 1. Each
    // carries the accumulator offset of its target relative to the input's staged position:
    // uid = id - (fid - centre) -> row y - oy, column z - oz, slice of channel oc.
    {
        int carry = 0;
        for (int g0 = 0; g0 < G; g0 += blockDim.x) {
            const int g = g0 + threadIdx.x;
            int cnt = 0;
            if (g < G) cnt = a.off2[g * (c_out + 1) + oc0 + nocl] - a.off2[g * (c_out + 1) + oc0];
            int tot;
            const int ex = block_excl_scan(cnt, reinterpret_cast<int*>(misc), &tot);
            if (g < G) swoff[g] = carry + ex;
            carry += tot;
        }
        if (threadIdx.x == 0) swoff[G] = carry;
        __syncthreads();
        for (int g = warp; g < G; g += kFwdWarps) {
            const int lo = a.off2[g * (c_out + 1) + oc0];
            const int n = swoff[g + 1] - swoff[g];
            const int oy = g % kg.ky - kg.hy;
            for (int j = lane; j < n; j += 32) {
                const int2 m = a.meta2[lo + j];
                sw4[swoff[g] + j] = make_int4((m.x - oc0) * TYZR - m.y + (ylo - y0 - oy) * ZR,
                                              __float_as_int(a.val2[lo + j]), oy, 0);
            }
        }
    }

    // ------------------------------------------------------------ accumulate (Alg. 1 inner loops)
    const int yw0 = y0 + warp * t.RW, yw1 = min(yw0 + t.RW, ye);
    const uint32_t nrw = (uint32_t)max(0, yw1 - yw0);
    const float invZ = 1.0f / (float)Z;
    // row pointers of every (ic, input plane), rows ylo..yhi, in one burst
    for (int q = threadIdx.x; q < PK * NRP; q += blockDim.x) {
        const int pk = q / NRP, r = q - pk * NRP;
        const int ic = pk / kg.kx, pl = pk - ic * kg.kx;
        const int xs = x + pl - kg.hx;
        rp[q] = (xs >= 0 && xs < gx.X) ? a.xrow[((b * c_in + ic) * gx.X + xs) * (int64_t)gx.Y + ylo + r] : 0u;
    }
    __syncthreads();
    {   // stage offsets of every (ic, plane) run
        int carry = 0;
        for (int p0 = 0; p0 < PK; p0 += blockDim.x) {
            const int pk = p0 + threadIdx.x;
            const int cnt = pk < PK ? (int)(rp[pk * NRP + nr] - rp[pk * NRP]) : 0;
            int tot;
            const int ex = block_excl_scan(cnt, reinterpret_cast<int*>(misc), &tot);
            if (pk < PK) sbase[pk] = carry + ex;
            carry += tot;
        }
        if (threadIdx.x == 0) sbase[PK] = carry;
        __syncthreads();
    }
    // chunks of input channels whose stored inputs fit the stage (one coalesced burst each)
    for (int ic0 = 0; ic0 < c_in;) {
        int ic1 = ic0 + 1;
        while (ic1 < c_in && sbase[(ic1 + 1) * kg.kx] - sbase[ic0 * kg.kx] <= kStageCap) ++ic1;
        const int sb0 = sbase[ic0 * kg.kx];
        const int nst = sbase[ic1 * kg.kx] - sb0;
        const bool staged = nst <= kStageCap;        // false only for one over-full channel
        if (staged) {
            // one warp per (ic, plane) run: coalesced loads, no per-entry search
            for (int pk = ic0 * kg.kx + warp; pk < ic1 * kg.kx; pk += kFwdWarps) {
                const int ic = pk / kg.kx, xs = x + (pk - ic * kg.kx) - kg.hx;
                const uint32_t g0 = rp[pk * NRP];
                const int n = sbase[pk + 1] - sbase[pk];
                uint2* dst = stage + (sbase[pk] - sb0);
                const uint64_t rowbase = (uint64_t)(((b * c_in + ic) * gx.X + xs) * (int64_t)gx.Y + ylo) * (uint64_t)Z;
                for (int i = lane; i < n; i += 32) {
                    const uint32_t L = (uint32_t)(a.xkeys[g0 + i] - rowbase);
                    const uint32_t yrel = div_small(L, (uint32_t)Z, invZ);
                    // {row (8 bits) | offset in the stage window (24 bits), value}
                    dst[i] = make_uint2((yrel << 24) | (yrel * (uint32_t)ZR + (L - yrel * (uint32_t)Z)),
                                        __float_as_uint(a.xvals[g0 + i]));
                }
            }
        }
        __syncthreads();
        // work items (ic, input plane): the inputs of rows yw0-hy .. yw1+hy against all weights of
        // (ic, dx) whose target row falls in this warp's rows
        const int pk1 = (yw0 < yw1) ? ic1 * kg.kx : 0;
        for (int pk = ic0 * kg.kx; pk < pk1; ++pk) {
            const uint32_t* RP = rp + pk * NRP;
            const int r0 = max(ylo, yw0 - kg.hy) - ylo, r1 = min(yhi, yw1 + kg.hy) - ylo;
            const uint32_t e0 = RP[r0], e1 = RP[r1];
            if (e0 == e1) continue;
            const int wlo = swoff[pk * kg.ky], whi = swoff[(pk + 1) * kg.ky];
            if (wlo == whi) continue;
            const int n = (int)(e1 - e0);
            const int s0 = staged ? sbase[pk] - sb0 + (int)(e0 - RP[0]) : 0;
            uint64_t rowbase = 0;
            if (!staged) {
                const int ic = pk / kg.kx, xs = x + (pk - ic * kg.kx) - kg.hx;
                rowbase = (uint64_t)(((b * c_in + ic) * gx.X + xs) * (int64_t)gx.Y + ylo) * (uint64_t)Z;
            }
            for (int c = 0; c < n; c += 32) {
                const bool valid = c + lane < n;
                int pos = 0, rel = -1000;                     // rel: input row - yw0
                float v = 0.0f;
                if (valid) {
                    uint32_t yrel;
                    if (staged) {
                        const uint2 en = stage[s0 + c + lane];
                        pos = (int)(en.x & 0xffffffu);
                        v = __uint_as_float(en.y);
                        yrel = en.x >> 24;
                    } else {
                        const uint32_t L = (uint32_t)(a.xkeys[e0 + c + lane] - rowbase);
                        yrel = div_small(L, (uint32_t)Z, invZ);
                        pos = (int)(yrel * (uint32_t)ZR + (L - yrel * (uint32_t)Z));
                        v = a.xvals[e0 + c + lane];
                    }
                    rel = ylo + (int)yrel - yw0;
                }
                for (int j = wlo; j < whi; ++j) {
                    const int4 q = sw4[j];
                    const int wd = q.x;
                    const float w = __int_as_float(q.y);
                    // target row (input row - oy) must be one of this warp's rows
                    if ((uint32_t)(rel - q.z) < nrw) {
#ifdef SPC_DEBUG
                        if (pos + wd < -t.pad || pos + wd >= t.ocg * TYZR + t.pad)
                            printf("OOB b=%lld x=%d ty=%d oc0=%d warp=%d lane=%d pk=%d pos=%d wd=%d j=%d\n",
                                   (long long)b, x, ty, oc0, warp, lane, pk, pos, wd, j);
#endif
                        // "add val*fval to buffer at uid"
                        float* p = acc + pos + wd;
                        const float old = *p;
                        const float base = __float_as_uint(old) == kAbsent ? 0.0f : old;
                        *p = fmaf(v, w, base);
                    }
                    __syncwarp();   // the next weight's lanes may read what this step wrote
                }
            }
        }
        __syncthreads();                                 // stage consumed
        ic0 = ic1;
    }

    // ------------------------------------------------------------------------ epilogue
    // "get non-zero entries" and "add bias to non-zero entries": the tile's slice
    // of the pre-attention responses goes to the (b, oc) buffers -- the paper's temporary dense
    // buffer, absent marker where there is no support -- while the support size and a
    // histogram of the top score digit are accumulated for the attention threshold.
    const int nyr = ye - y0;
    const bool do_hist = a.attn != SPC_ATTN_NONE;
    for (int ocl = 0; ocl < nocl; ++ocl) {
        const int oc = oc0 + ocl;
        const int64_t s = b * c_out + oc;
        const float bv = a.bias ? a.bias[oc] : 0.0f;
        const float* A = acc + ocl * TYZR;
        if (do_hist)
            for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        uint32_t cnt = 0;
        float* P = a.pre + s * gy.V + ((int64_t)x * gy.Y + y0) * Z;
        const bool vec = (Z & 3) == 0;
        for (int r = warp; r < nyr; r += kFwdWarps) {
            for (int z0 = 4 * lane; z0 < Z; z0 += 128) {
                float v[4];
                if (vec) {
                    const float4 q = *reinterpret_cast<const float4*>(A + r * ZR + z0);
                    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[u] = z0 + u < Z ? A[r * ZR + z0 + u] : __uint_as_float(kAbsent);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (__float_as_uint(v[u]) != kAbsent) {
                        v[u] += bv;
                        ++cnt;
                        if (do_hist) atomicAdd(&hist[score_bits(__float_as_uint(v[u]), a.attn) >> 21], 1u);
                    }
                }
                if (vec) {
                    __stcs(reinterpret_cast<float4*>(P + (int64_t)r * Z + z0), make_float4(v[0], v[1], v[2], v[3]));
                } else {
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (z0 + u < Z) __stcs(P + (int64_t)r * Z + z0 + u, v[u]);
                }
            }
        }
        const uint32_t tot = block_sum(cnt, misc);
        if (threadIdx.x == 0 && tot) atomicAdd(&a.seg_count[s], (unsigned long long)tot);
        if (do_hist)
            for (int i = threadIdx.x; i < kSelBins; i += blockDim.x)
                if (hist[i]) atomicAdd(&a.hist[s * kSelBins + i], hist[i]);
        __syncthreads();
    }
}

// ------------------------------------------------------------------- per-segment kernels
// find: threshold digit B1 (bins scanned from the top until the count reaches k).
__global__ void fwd_find_kernel(FwdArgs a, int64_t nseg) {
    const int64_t s = blockIdx.x;
    __shared__ uint64_t sm[33];
    const int64_t n = (int64_t)a.seg_count[s];
    FwdSeg st{};
    const bool keep_all = a.attn == SPC_ATTN_NONE || n <= a.k;
    if (keep_all) {
        if (threadIdx.x == 0) {
            st.keep_all = 1;
            st.kstar = 0;
            a.seg[s] = st;
            a.cand_cnt[s] = 0;
        }
        return;
    }
    const uint32_t* h = a.hist + s * kSelBins;
    constexpr int per = kSelBins / 256;
    uint64_t local = 0;
    for (int q = 0; q < per; ++q) local += h[kSelBins - 1 - threadIdx.x * per - q];
    uint64_t tot;
    const uint64_t before = block_excl_scan(local, sm, &tot);
    const uint64_t need = (uint64_t)a.k;
    if (before < need && before + local >= need) {
        uint64_t cum = before;
        for (int q = 0; q < per; ++q) {
            const int bin = kSelBins - 1 - threadIdx.x * per - q;
            if (cum + h[bin] >= need) {
                st.keep_all = 0;
                st.b1 = (uint32_t)bin;
                st.need = (int64_t)(need - cum);
                st.kstar = 0;
                a.seg[s] = st;
                a.cand_cnt[s] = h[bin];
                break;
            }
            cum += h[bin];
        }
    }
}

// exclusive scan of a per-segment u64 array (single block); total -> *total
__global__ void seg_scan_u64_kernel(const uint64_t* in, uint64_t* out, int64_t n, int64_t* total) {
    __shared__ uint64_t sm[33];
    uint64_t carry = 0;
    for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const uint64_t v = i < n ? in[i] : 0;
        uint64_t t;
        const uint64_t ex = block_excl_scan(v, sm, &t);
        if (i < n) out[i] = carry + ex;
        carry += t;
    }
    if (threadIdx.x == 0) {
        out[n] = carry;
        if (total) *total = (int64_t)carry;
    }
}

constexpr int kChunkThreads = 256;
constexpr int kChunkItems = 16;
constexpr int kChunk = kChunkThreads * kChunkItems;   // voxels per chunk of a (b, oc) buffer

// classify (HBM stream over the buffers): per chunk the entries kept outright (digit > B1, or
// every support entry when the segment keeps all) and the candidates (digit == B1), which are
// appended to the segment's candidate list.
__global__ void __launch_bounds__(kChunkThreads) fwd_classify_kernel(FwdArgs a, int64_t V) {
    const int64_t s = blockIdx.x / a.nchunk, c = blockIdx.x % a.nchunk;
    const FwdSeg st = a.seg[s];
    const int64_t lo = c * kChunk;
    const float* P = a.pre + s * V;
    __shared__ uint32_t sh_cnt, sh_base, sh_slot;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) { sh_cnt = 0; sh_slot = 0; }
    // element u of this thread: lo + 4*(v*256 + tid) + w, u = 4v + w (float4 loads, coalesced)
    uint32_t bits[kChunkItems];
    const bool vec = (V & 3) == 0;
#pragma unroll
    for (int v = 0; v < kChunkItems / 4; ++v) {
        const int64_t i = lo + 4 * ((int64_t)v * kChunkThreads + threadIdx.x);
        if (vec && i + 4 <= V) {
            const float4 q = __ldcs(reinterpret_cast<const float4*>(P + i));
            bits[4 * v] = __float_as_uint(q.x);
            bits[4 * v + 1] = __float_as_uint(q.y);
            bits[4 * v + 2] = __float_as_uint(q.z);
            bits[4 * v + 3] = __float_as_uint(q.w);
        } else {
#pragma unroll
            for (int w = 0; w < 4; ++w) bits[4 * v + w] = i + w < V ? __float_as_uint(P[i + w]) : kAbsent;
        }
    }
    uint32_t packed = 0;   // kept outright (low 16 bits) | candidates (high 16 bits)
#pragma unroll
    for (int u = 0; u < kChunkItems; ++u) {
        if (bits[u] == kAbsent) continue;
        if (st.keep_all) { ++packed; continue; }
        const uint32_t d = score_bits(bits[u], a.attn) >> 21;
        packed += (d > st.b1) + ((uint32_t)(d == st.b1) << 16);
    }
    packed = warp_sum(packed);
    __syncthreads();
    if (lane == 0 && packed) atomicAdd(&sh_cnt, packed);
    __syncthreads();
    const uint32_t tot = sh_cnt;
    const uint32_t tcand = tot >> 16;
    if (threadIdx.x == 0) {
        a.tile_def[s * a.nchunk + c] = tot & 0xffffu;
        sh_base = tcand ? (uint32_t)atomicAdd(&a.cand_cur[s], (unsigned long long)tcand) : 0u;
    }
    __syncthreads();
    if (tcand == 0) return;
    const uint64_t base = a.cand_off[s] + sh_base;
#pragma unroll
    for (int u = 0; u < kChunkItems; ++u) {
        const bool is_c = bits[u] != kAbsent && (score_bits(bits[u], a.attn) >> 21) == st.b1;
        const unsigned m = __ballot_sync(kFull, is_c);
        if (!m) continue;
        uint32_t slot0 = 0;
        if (lane == 0) slot0 = atomicAdd(&sh_slot, (uint32_t)__popc(m));
        slot0 = __shfl_sync(kFull, slot0, 0);
        if (is_c) {
            const uint32_t p = (uint32_t)(lo + 4 * ((int64_t)(u >> 2) * kChunkThreads + threadIdx.x) + (u & 3));
            a.cand[base + slot0 + __popc(m & ((1u << lane) - 1u))] = make_uint2(p, bits[u]);
        }
    }
}

// resolve: the `need` largest composite keys among the candidates of a segment (8-bit radix
// select over 64 bits, all keys distinct) -> kstar; then count selected candidates per chunk.
__global__ void __launch_bounds__(512) fwd_resolve_kernel(FwdArgs a) {
    const int64_t s = blockIdx.x;
    FwdSeg st = a.seg[s];
    if (st.keep_all) return;
    const uint64_t n = a.cand_cnt[s];
    const uint2* c = a.cand + a.cand_off[s];
    __shared__ uint32_t h[256];
    __shared__ uint64_t sh_prefix, sh_mask;
    __shared__ int64_t sh_need;
    if (threadIdx.x == 0) {
        sh_prefix = 0;
        sh_mask = 0;
        sh_need = st.need;
    }
    __syncthreads();
    for (int sh = 56; sh >= 0; sh -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
        __syncthreads();
        const uint64_t prefix = sh_prefix, mask = sh_mask;
        for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
            const uint2 e = c[i];
            const uint64_t k = composite(score_bits(e.y, a.attn), e.x);
            if ((k & mask) == prefix) atomicAdd(&h[(k >> sh) & 255], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            // warp scan of the 256 bins from the top: lane l owns bins 255-8l .. 248-8l
            const int l = threadIdx.x;
            uint32_t own = 0;
            for (int q = 0; q < 8; ++q) own += h[255 - 8 * l - q];
            const uint32_t incl = warp_incl_scan(own);
            const int64_t need = sh_need;
            const int64_t before = (int64_t)(incl - own);
            if (before < need && before + (int64_t)own >= need) {
                int64_t cum = before;
                for (int q = 0; q < 8; ++q) {
                    const int bin = 255 - 8 * l - q;
                    if (cum + (int64_t)h[bin] >= need) {
                        sh_need = need - cum;
                        sh_prefix = prefix | ((uint64_t)bin << sh);
                        sh_mask = mask | ((uint64_t)255 << sh);
                        break;
                    }
                    cum += h[bin];
                }
            }
        }
        __syncthreads();
    }
    const uint64_t kstar = sh_prefix;
    if (threadIdx.x == 0) {
        st.kstar = kstar;
        a.seg[s] = st;
    }
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint2 e = c[i];
        if (composite(score_bits(e.y, a.attn), e.x) >= kstar) atomicAdd(&a.tile_sel[s * a.nchunk + e.x / kChunk], 1u);
    }
}

// per segment: kept count per chunk -> exclusive offsets; segment total -> kept[s]
__global__ void fwd_chunk_scan_kernel(FwdArgs a, uint64_t* kept) {
    const int64_t s = blockIdx.x;
    __shared__ uint64_t sm[33];
    uint64_t carry = 0;
    for (int64_t base = 0; base < a.nchunk; base += blockDim.x) {
        const int64_t c = base + threadIdx.x;
        uint64_t v = 0;
        if (c < a.nchunk) v = (uint64_t)a.tile_def[s * a.nchunk + c] + a.tile_sel[s * a.nchunk + c];
        uint64_t tot;
        const uint64_t ex = block_excl_scan(v, sm, &tot);
        if (c < a.nchunk) a.tile_off[s * a.nchunk + c] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) kept[s] = carry;
}

// write (HBM stream): keep iff composite(score, p) >= kstar (all support when keep-all);
// ordered compaction in key order ("compress ids ... write k largest features").
__global__ void __launch_bounds__(kChunkThreads) fwd_write_kernel(FwdArgs a, int64_t V) {
    const int64_t s = blockIdx.x / a.nchunk, c = blockIdx.x % a.nchunk;
    const FwdSeg st = a.seg[s];
    const int64_t lo = c * kChunk + (int64_t)threadIdx.x * kChunkItems;
    const float* P = a.pre + s * V;
    __shared__ uint64_t sm[33];
    uint32_t bits[kChunkItems];
    uint32_t keep = 0;
    if (lo + kChunkItems <= V && (V & 3) == 0) {
#pragma unroll
        for (int u = 0; u < kChunkItems; u += 4) {
            const float4 q = __ldcs(reinterpret_cast<const float4*>(P + lo + u));
            bits[u] = __float_as_uint(q.x);
            bits[u + 1] = __float_as_uint(q.y);
            bits[u + 2] = __float_as_uint(q.z);
            bits[u + 3] = __float_as_uint(q.w);
        }
    } else {
#pragma unroll
        for (int u = 0; u < kChunkItems; ++u) bits[u] = lo + u < V ? __float_as_uint(P[lo + u]) : kAbsent;
    }
#pragma unroll
    for (int u = 0; u < kChunkItems; ++u) {
        bool k = bits[u] != kAbsent;
        if (k && !st.keep_all) k = composite(score_bits(bits[u], a.attn), (uint32_t)(lo + u)) >= st.kstar;
        keep |= (uint32_t)k << u;
    }
    uint64_t tot;
    uint64_t pos = a.seg_off[s] + a.tile_off[s * a.nchunk + c] + block_excl_scan((uint64_t)__popc(keep), sm, &tot);
#pragma unroll
    for (int u = 0; u < kChunkItems; ++u) {
        if (keep & (1u << u)) {
            a.out_keys[pos] = (uint64_t)s * (uint64_t)V + (uint64_t)(lo + u);
            a.out_vals[pos] = __uint_as_float(bits[u]);
            ++pos;
        }
    }
}

cudaError_t launch_conv_fwd_pipeline(const Geo& gx, const Geo& gy, const KGeo& kg, const FwdTile& t,
                                     const FwdArgs& a, cudaStream_t s) {
    const int64_t nseg = gy.B * gy.C;
    if (nseg == 0) return cudaMemsetAsync(a.out_nnz, 0, sizeof(int64_t), s);
    cudaError_t e = cudaFuncSetAttribute(conv_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t.smem);
    if (e != cudaSuccess) return e;
    const size_t segb = sizeof(uint64_t) * (size_t)nseg;
    cudaMemsetAsync(a.seg_count, 0, segb, s);
    cudaMemsetAsync(a.cand_cur, 0, segb, s);
    cudaMemsetAsync(a.tile_sel, 0, sizeof(uint32_t) * (size_t)(nseg * a.nchunk), s);
    if (a.attn != SPC_ATTN_NONE) cudaMemsetAsync(a.hist, 0, sizeof(uint32_t) * kSelBins * (size_t)nseg, s);
    const dim3 grid((unsigned)(gy.B * gy.X * t.nty), (unsigned)t.n_ocg);
    const unsigned sgrid = (unsigned)(nseg * a.nchunk);
    { SPC_PHASE("conv_fwd", s, 1); conv_fwd_kernel<<<grid, kFwdThreads, t.smem, s>>>(gx, gy, kg, t, a); }
    { SPC_PHASE("fwd_find", s, 1); fwd_find_kernel<<<(unsigned)nseg, 256, 0, s>>>(a, nseg); }
    if (a.attn != SPC_ATTN_NONE) {
        SPC_PHASE("seg_scan", s, 1);
        seg_scan_u64_kernel<<<1, 1024, 0, s>>>(a.cand_cnt, a.cand_off, nseg, nullptr);
    }
    { SPC_PHASE("fwd_classify", s, 1); fwd_classify_kernel<<<sgrid, kChunkThreads, 0, s>>>(a, gy.V); }
    if (a.attn != SPC_ATTN_NONE) {
        SPC_PHASE("fwd_resolve", s, 1);
        fwd_resolve_kernel<<<(unsigned)nseg, 512, 0, s>>>(a);
    }
    // kept per segment goes to cand_cnt (reused as scratch), then segment offsets
    { SPC_PHASE("fwd_chunk_scan", s, 1); fwd_chunk_scan_kernel<<<(unsigned)nseg, 256, 0, s>>>(a, a.cand_cnt); }
    { SPC_PHASE("seg_scan", s, 1); seg_scan_u64_kernel<<<1, 1024, 0, s>>>(a.cand_cnt, a.seg_off, nseg, a.out_nnz); }
    { SPC_PHASE("fwd_write", s, 1); fwd_write_kernel<<<sgrid, kChunkThreads, 0, s>>>(a, gy.V); }
    return cudaGetLastError();
}

}  // namespace spc

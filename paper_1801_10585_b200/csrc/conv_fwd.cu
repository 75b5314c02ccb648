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
constexpr size_t kFwdBudget = 110 * 1024;   // two CTAs per SM
constexpr int kStageCap = 2048;             // staged input entries per input channel

// shared-memory bytes beyond the accumulator
static size_t fwd_fixed_smem(const KGeo& kg, int c_in, int TY, int64_t nwg) {
    const size_t nrp = (size_t)c_in * kg.kx * (TY + 2 * kg.hy + 1);
    return (size_t)kSelBins * 4 + 256 * 4 + (size_t)nwg * 8 + (size_t)(c_in * kg.kx * kg.ky + 1) * 4 + nrp * 4 +
           (size_t)(c_in * kg.kx + 1) * 4 + 16 + (size_t)kStageCap * 8 + 64;
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
    TY = std::min(TY, gy.Y);
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

template <int MODE>
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
    const int ti = x * t.nty + ty;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int TYZR = t.TY * ZR;

    // layout: [pad][acc ocg*TY*ZR][pad] | hist | misc(256) | swd | sww | swoff | rp | sbase | stage
    const int KXY = kg.kx * kg.ky;
    const int G = c_in * KXY;
    const int ylo = max(0, y0 - kg.hy), yhi = min(gy.Y, ye + kg.hy);
    const int nr = yhi - ylo;                        // input rows read per plane
    float* acc = smf + t.pad;
    uint32_t* hist = reinterpret_cast<uint32_t*>(smf + 2 * t.pad + t.ocg * TYZR);
    uint32_t* misc = hist + kSelBins;
    int* swd = reinterpret_cast<int*>(misc + 256);   // group weights: acc offset (ocl*TY*ZR - oz)
    float* sww = reinterpret_cast<float*>(swd + t.nwg_max);
    int* swoff = reinterpret_cast<int*>(sww + t.nwg_max);
    uint32_t* rp = reinterpret_cast<uint32_t*>(swoff + G + 1);
    const int PK = c_in * kg.kx;                     // (input channel, input plane) pairs
    int* sbase = reinterpret_cast<int*>(rp + PK * (t.TY + 2 * kg.hy + 1));
    uint2* stage = reinterpret_cast<uint2*>((reinterpret_cast<uintptr_t>(sbase + PK + 1) + 15) & ~(uintptr_t)15);

    {
        const int n4 = (2 * t.pad + t.ocg * TYZR) / 4;
        uint4 ab = make_uint4(kAbsent, kAbsent, kAbsent, kAbsent);
        for (int i = threadIdx.x; i < n4; i += blockDim.x) reinterpret_cast<uint4*>(smf)[i] = ab;
    }
    // this group's weights, grouped by (ic, dx, dy): "filter(oc, ic)" of Alg. 1
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
            for (int j = lane; j < n; j += 32) {
                const int2 m = a.meta2[lo + j];
                swd[swoff[g] + j] = (m.x - oc0) * TYZR - m.y;
                sww[swoff[g] + j] = a.val2[lo + j];
            }
        }
    }

    // ------------------------------------------------------------ accumulate (Alg. 1 inner loops)
    const int yw0 = y0 + warp * t.RW, yw1 = min(yw0 + t.RW, ye);
    const float invZ = 1.0f / (float)Z;
    const int NRP = nr + 1;
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
            for (int i = threadIdx.x; i < nst; i += blockDim.x) {
                const int gi = sb0 + i;
                int lo = ic0 * kg.kx, hi = ic1 * kg.kx - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (sbase[mid] <= gi) lo = mid; else hi = mid - 1;
                }
                const int ic = lo / kg.kx, pl = lo - ic * kg.kx;
                const uint32_t ge = rp[lo * NRP] + (uint32_t)(gi - sbase[lo]);
                const int xs = x + pl - kg.hx;
                const uint64_t rowbase = (uint64_t)(((b * c_in + ic) * gx.X + xs) * (int64_t)gx.Y + ylo) * (uint64_t)Z;
                const uint32_t L = (uint32_t)(a.xkeys[ge] - rowbase);
                const uint32_t yrel = div_small(L, (uint32_t)Z, invZ);
                stage[i] = make_uint2(yrel * (uint32_t)ZR + (L - yrel * (uint32_t)Z), __float_as_uint(a.xvals[ge]));
            }
        }
        __syncthreads();
        for (int ic = ic0; ic < ic1 && yw0 < yw1; ++ic)
        for (int dxy = 0; dxy < KXY; ++dxy) {
            const int pl = dxy / kg.ky, oy = dxy - pl * kg.ky - kg.hy;
            const int xs = x + pl - kg.hx;                   // input plane of uid_x = x
            if (xs < 0 || xs >= gx.X) continue;
            const int g = ic * KXY + dxy;
            const int w0 = swoff[g], nwt = swoff[g + 1] - w0;
            if (nwt == 0) continue;
            const int yr0 = max(ylo, yw0 + oy), yr1 = min(yhi, yw1 + oy);
            if (yr0 >= yr1) continue;
            const int pk = ic * kg.kx + pl;
            const uint32_t* RP = rp + pk * NRP;
            const uint32_t e0 = RP[yr0 - ylo], e1 = RP[yr1 - ylo];
            if (e0 == e1) continue;
            const int shift = (ylo - y0 - oy) * ZR;           // input row offset -> target row offset
            const int n = (int)(e1 - e0);
            const int s0 = staged ? sbase[pk] - sb0 + (int)(e0 - RP[0]) : 0;
            const uint64_t rowbase = (uint64_t)(((b * c_in + ic) * gx.X + xs) * (int64_t)gx.Y + ylo) * (uint64_t)Z;
            for (int c = 0; c < n; c += 32) {
                const bool valid = c + lane < n;
                int pos = 0;
                float v = 0.0f;
                if (valid) {
                    if (staged) {
                        const uint2 en = stage[s0 + c + lane];
                        pos = (int)en.x;
                        v = __uint_as_float(en.y);
                    } else {
                        const uint32_t L = (uint32_t)(a.xkeys[e0 + c + lane] - rowbase);
                        const uint32_t yrel = div_small(L, (uint32_t)Z, invZ);
                        pos = (int)(yrel * (uint32_t)ZR + (L - yrel * (uint32_t)Z));
                        v = a.xvals[e0 + c + lane];
                    }
                    pos += shift;
                }
                for (int j = 0; j < nwt; ++j) {
                    const int wd = swd[w0 + j];
                    const float w = sww[w0 + j];
#ifdef SPC_DEBUG
                    if (valid && (pos + wd < -t.pad || pos + wd >= t.ocg * TYZR + t.pad))
                        printf("OOB b=%lld x=%d ty=%d oc0=%d warp=%d lane=%d ic=%d dxy=%d pos=%d wd=%d j=%d w0=%d "
                               "nwt=%d shift=%d s0=%d c=%d yr0=%d yr1=%d e0=%u e1=%u staged=%d swoffG=%d\n",
                               (long long)b, x, ty, oc0, warp, lane, ic, dxy, pos, wd, j, w0, nwt, shift, s0, c, yr0,
                               yr1, e0, e1, (int)staged, swoff[G]);
#endif
                    if (valid) {
                        // "add val*fval to buffer at uid", uid = id - (fid - centre)
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

    // ------------------------------------------------------------------------ epilogues
    const int nyr = ye - y0;
    const int nvox = nyr * Z;
    for (int ocl = 0; ocl < nocl; ++ocl) {
        const int oc = oc0 + ocl;
        const int64_t s = b * c_out + oc;
        const float bv = a.bias ? a.bias[oc] : 0.0f;
        const float* A = acc + ocl * TYZR;
        if (MODE == 0) {
            // support count + histogram of the top score digit ("get non-zero entries",
            // "add bias")
            const bool do_hist = a.attn != SPC_ATTN_NONE;
            if (do_hist)
                for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) hist[i] = 0;
            __syncthreads();
            uint32_t cnt = 0;
            for (int r = warp; r < nyr; r += kFwdWarps) {
                for (int z = lane; z < Z; z += 32) {
                    const float v = A[r * ZR + z];
                    if (__float_as_uint(v) == kAbsent) continue;
                    ++cnt;
                    if (do_hist) atomicAdd(&hist[score_bits(__float_as_uint(v + bv), a.attn) >> 21], 1u);
                }
            }
            const uint32_t tot = block_sum(cnt, misc);
            if (threadIdx.x == 0) {
                a.tile_cnt[s * t.NT + ti] = tot;
                if (tot) atomicAdd(&a.seg_count[s], (unsigned long long)tot);
            }
            if (do_hist)
                for (int i = threadIdx.x; i < kSelBins; i += blockDim.x)
                    if (hist[i]) atomicAdd(&a.hist[s * kSelBins + i], hist[i]);
            __syncthreads();
        } else if (MODE == 1) {
            const FwdSeg st = a.seg[s];
            if (st.keep_all) continue;                   // uniform over the block
            uint32_t ndef = 0, ncand = 0;
            for (int r = warp; r < nyr; r += kFwdWarps) {
                for (int z = lane; z < Z; z += 32) {
                    const float v = A[r * ZR + z];
                    if (__float_as_uint(v) == kAbsent) continue;
                    const uint32_t d = score_bits(__float_as_uint(v + bv), a.attn) >> 21;
                    ndef += d > st.b1;
                    ncand += d == st.b1;
                }
            }
            const uint32_t tdef = block_sum(ndef, misc);
            const uint32_t tcand = block_sum(ncand, misc);
            if (threadIdx.x == 0) {
                a.tile_def[s * t.NT + ti] = tdef;
                misc[40] = tcand ? (uint32_t)atomicAdd(&a.cand_cur[s], (unsigned long long)tcand) : 0u;
                misc[41] = 0;
            }
            __syncthreads();
            if (tcand) {
                const uint64_t base = a.cand_off[s] + misc[40];
                for (int r = warp; r < nyr; r += kFwdWarps) {
                    for (int z = lane; z < Z; z += 32) {
                        const float v = A[r * ZR + z];
                        if (__float_as_uint(v) == kAbsent) continue;
                        const float val = v + bv;
                        if ((score_bits(__float_as_uint(val), a.attn) >> 21) != st.b1) continue;
                        const uint32_t slot = atomicAdd(&misc[41], 1u);
                        const uint32_t p = (uint32_t)(((int64_t)x * gy.Y + (y0 + r)) * Z + z);
                        a.cand[base + slot] = make_uint2(p, __float_as_uint(val));
                    }
                }
            }
            __syncthreads();
        } else {
            // keep iff composite(score, p) >= kstar; ordered compaction in key order
            const FwdSeg st = a.seg[s];
            const int per = (nvox + kFwdThreads - 1) / kFwdThreads;
            const int l0 = threadIdx.x * per, l1 = min(l0 + per, nvox);
            const uint32_t pbase = (uint32_t)(((int64_t)x * gy.Y + y0) * Z);
            uint32_t nk = 0;
            {
                int r = l0 / Z, z = l0 - (l0 / Z) * Z;
                for (int l = l0; l < l1; ++l) {
                    const float v = A[r * ZR + z];
                    if (__float_as_uint(v) != kAbsent) {
                        const uint32_t sc = score_bits(__float_as_uint(v + bv), a.attn);
                        nk += st.keep_all || composite(sc, pbase + (uint32_t)l) >= st.kstar;
                    }
                    if (++z == Z) { z = 0; ++r; }
                }
            }
            uint32_t tot;
            uint64_t pos = a.seg_off[s] + a.tile_off[s * t.NT + ti] + block_excl_scan(nk, misc, &tot);
            if (nk) {
                int r = l0 / Z, z = l0 - (l0 / Z) * Z;
                for (int l = l0; l < l1; ++l) {
                    const float v = A[r * ZR + z];
                    if (__float_as_uint(v) != kAbsent) {
                        const float val = v + bv;
                        const uint32_t sc = score_bits(__float_as_uint(val), a.attn);
                        if (st.keep_all || composite(sc, pbase + (uint32_t)l) >= st.kstar) {
                            a.out_keys[pos] = (uint64_t)s * (uint64_t)gy.V + pbase + (uint32_t)l;
                            a.out_vals[pos] = val;
                            ++pos;
                        }
                    }
                    if (++z == Z) { z = 0; ++r; }
                }
            }
        }
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

// resolve: the `need` largest composite keys among the candidates of a segment (8-bit radix
// select over 64 bits, all keys distinct) -> kstar; then count selected candidates per tile.
__global__ void __launch_bounds__(512) fwd_resolve_kernel(FwdArgs a, Geo gy, FwdTile t) {
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
        if (threadIdx.x == 0) {
            int64_t need = sh_need, cum = 0;
            for (int bin = 255; bin >= 0; --bin) {
                if (cum + (int64_t)h[bin] >= need) {
                    sh_need = need - cum;
                    sh_prefix = prefix | ((uint64_t)bin << sh);
                    sh_mask = mask | ((uint64_t)255 << sh);
                    break;
                }
                cum += h[bin];
            }
        }
        __syncthreads();
    }
    const uint64_t kstar = sh_prefix;
    if (threadIdx.x == 0) {
        st.kstar = kstar;
        a.seg[s] = st;
    }
    const uint32_t YZ = (uint32_t)gy.Y * (uint32_t)gy.Z;
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint2 e = c[i];
        if (composite(score_bits(e.y, a.attn), e.x) >= kstar) {
            const uint32_t px = e.x / YZ, py = (e.x / (uint32_t)gy.Z) % (uint32_t)gy.Y;
            atomicAdd(&a.tile_sel[s * t.NT + px * t.nty + py / t.TY], 1u);
        }
    }
}

// per segment: kept count per tile -> exclusive offsets; segment total -> kept[s]
__global__ void fwd_tile_scan_kernel(FwdArgs a, FwdTile t, uint64_t* kept) {
    const int64_t s = blockIdx.x;
    const FwdSeg st = a.seg[s];
    __shared__ uint64_t sm[33];
    uint64_t carry = 0;
    for (int base = 0; base < t.NT; base += blockDim.x) {
        const int ti = base + threadIdx.x;
        uint64_t v = 0;
        if (ti < t.NT)
            v = st.keep_all ? a.tile_cnt[s * t.NT + ti] : (uint64_t)a.tile_def[s * t.NT + ti] + a.tile_sel[s * t.NT + ti];
        uint64_t tot;
        const uint64_t ex = block_excl_scan(v, sm, &tot);
        if (ti < t.NT) a.tile_off[s * t.NT + ti] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0) kept[s] = carry;
}

cudaError_t launch_conv_fwd_pipeline(const Geo& gx, const Geo& gy, const KGeo& kg, const FwdTile& t,
                                     const FwdArgs& a, cudaStream_t s) {
    const int64_t nseg = gy.B * gy.C;
    if (nseg == 0) return cudaMemsetAsync(a.out_nnz, 0, sizeof(int64_t), s);
    cudaError_t e;
    e = cudaFuncSetAttribute(conv_fwd_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t.smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(conv_fwd_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t.smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(conv_fwd_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t.smem);
    if (e != cudaSuccess) return e;
    const size_t segb = sizeof(uint64_t) * (size_t)nseg;
    cudaMemsetAsync(a.seg_count, 0, segb, s);
    cudaMemsetAsync(a.cand_cur, 0, segb, s);
    cudaMemsetAsync(a.tile_sel, 0, sizeof(uint32_t) * (size_t)nseg * t.NT, s);
    if (a.attn != SPC_ATTN_NONE) cudaMemsetAsync(a.hist, 0, sizeof(uint32_t) * kSelBins * (size_t)nseg, s);
    const dim3 grid((unsigned)(gy.B * gy.X * t.nty), (unsigned)t.n_ocg);
    { SPC_PHASE("conv_fwd_hist", s, 1); conv_fwd_kernel<0><<<grid, kFwdThreads, t.smem, s>>>(gx, gy, kg, t, a); }
    { SPC_PHASE("fwd_find", s, 1); fwd_find_kernel<<<(unsigned)nseg, 256, 0, s>>>(a, nseg); }
    if (a.attn != SPC_ATTN_NONE) {
        { SPC_PHASE("seg_scan", s, 1); seg_scan_u64_kernel<<<1, 1024, 0, s>>>(a.cand_cnt, a.cand_off, nseg, nullptr); }
        { SPC_PHASE("conv_fwd_classify", s, 1); conv_fwd_kernel<1><<<grid, kFwdThreads, t.smem, s>>>(gx, gy, kg, t, a); }
        { SPC_PHASE("fwd_resolve", s, 1); fwd_resolve_kernel<<<(unsigned)nseg, 512, 0, s>>>(a, gy, t); }
    }
    // kept per segment goes to cand_cnt (reused as scratch), then segment offsets
    { SPC_PHASE("fwd_tile_scan", s, 1); fwd_tile_scan_kernel<<<(unsigned)nseg, 256, 0, s>>>(a, t, a.cand_cnt); }
    { SPC_PHASE("seg_scan", s, 1); seg_scan_u64_kernel<<<1, 1024, 0, s>>>(a.cand_cnt, a.seg_off, nseg, a.out_nnz); }
    { SPC_PHASE("conv_fwd_write", s, 1); conv_fwd_kernel<2><<<grid, kFwdThreads, t.smem, s>>>(gx, gy, kg, t, a); }
    return cudaGetLastError();
}

}  // namespace spc

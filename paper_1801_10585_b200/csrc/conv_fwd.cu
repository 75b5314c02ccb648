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
constexpr size_t kFwdBudget = 113 * 1024;   // two CTAs (16 warps) per SM
constexpr int kRing = 4;                    // per-warp cp.async ring: jobs in flight
constexpr int kRingSlotB = 32 * 8;          // one item: 32 key low words + 32 values
constexpr int kRingWords = kFwdWarps * kRing * kRingSlotB / 4 > kSelBins + 32 ? kFwdWarps * kRing * kRingSlotB / 4
                                                                              : kSelBins + 32;
static_assert(kRingWords >= kSelBins + 32, "the epilogue histogram (+ 32 dummy bins) reuses the ring");

static size_t r4(size_t n) { return (n + 3) & ~(size_t)3; }

// shared-memory bytes beyond the accumulator
static size_t fwd_fixed_smem(const KGeo& kg, int c_in, int TY, int64_t nwg) {
    const size_t PK = (size_t)c_in * kg.kx;
    return 4 * (512 + 4 * (size_t)nwg + 2 * r4(PK + 1) + r4(PK * (TY + 2 * kg.hy + 1)) + (size_t)kRingWords) + 64;
}

FwdTile plan_fwd_tile(const Geo& gy, const KGeo& kg, int c_out, int c_in, int64_t nw_total) {
    FwdTile t{};
    const int ZR = ((gy.Z + 2 * kg.hz + 3) / 4) * 4;
    const int pad = ((kg.hz + 3) / 4) * 4;
    const size_t row_b = (size_t)ZR * sizeof(float);
    auto rows = [&](int TY) { return TY + 2 * kg.hy + 2 * kg.hy * kFwdWarps; };
    auto need = [&](int ocg, int TY) {
        const int64_t nwg = std::min<int64_t>(nw_total, (int64_t)ocg * c_in * kg.KV);
        return fwd_fixed_smem(kg, c_in, TY, nwg) + (size_t)ocg * rows(TY) * row_b + (size_t)pad * 8;
    };
    // prefer >= 8 input rows per warp (lane utilisation), then the largest group of channels
    int TY = std::min(gy.Y, 8 * kFwdWarps);
    int ocg = std::min(c_out, 16);
    while (ocg > 1 && need(ocg, TY) > kFwdBudget) --ocg;
    while (TY > 1 && need(ocg, TY) > kFwdBudget) --TY;          // ocg == 1: shorter tiles
    if (need(ocg, TY) > kFwdBudget) { t.smem = 0; return t; }
    while (TY < gy.Y && need(ocg, TY + kFwdWarps) <= kFwdBudget) TY += kFwdWarps;   // spare room
    TY = std::min(TY, std::min(gy.Y, 240));   // staged rows are packed in 8 bits (TY + 2*hy < 256); TY <= 448 (row owners)
    t.TY = TY;
    t.RW = (TY + kFwdWarps - 1) / kFwdWarps;
    t.RT = rows(TY);
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

// The -0 accumulation mode of conv_fwd is exact iff every product of an input value and a weight
// is a nonzero multiple of 2^-149: true when all |x|, |w| >= 2^-50 (then no update can round to
// -0, the marker). This pass flags inputs that break it (weights: fwd_rounds_kernel).
__global__ void value_guard_kernel(const float* __restrict__ v, const int64_t* nnz_dev, int64_t bound,
                                   int* __restrict__ guard) {
    const int64_t n = load_n(nnz_dev, bound);
    bool bad = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float a = v[i];
        bad |= !(fabsf(a) >= 0x1p-50f) && !isnan(a);
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) *guard = 1;
}

// Weight rounds of one output-channel group (one block per group). Alg. 1 walks "for {fid,
// fval} in filter(oc, ic)"; the kernel below walks, per (ic, input plane dx), rounds that
// pair a weight of channel 2p with one of channel 2p+1: the two targets lie in different channel
// slices of the accumulator, so both read-modify-writes of a round can be in flight together.
// Round record {wdA, wA, wdB, wB}: wd = byte offset from an input's accumulator position to its
// target uid = id - (fid - centre) = slice(oc) - oy rows - oz columns. Per (ic, dx): first
// the two-channel rounds of every pair, then the leftovers of the longer list (wdB unused).
__global__ void fwd_rounds_kernel(KGeo kg, int c_in, int c_out, FwdTile t, const int2* __restrict__ meta2,
                                  const float* __restrict__ val2, const int* __restrict__ off2, int4* __restrict__ rec,
                                  int* __restrict__ pkoff, int* __restrict__ pkfull, int* __restrict__ guard) {
    __shared__ int sm[33];
    const int grp = blockIdx.x, oc0 = grp * t.ocg, nocl = min(t.ocg, c_out - oc0);
    const int PK = c_in * kg.kx, npair = (nocl + 1) / 2;
    const int SLb = t.RT * t.ZR * (int)sizeof(float);
    int4* R = rec + (int64_t)grp * t.nwg_max;
    int* PO = pkoff + (int64_t)grp * (PK + 1);
    int* PF = pkfull + (int64_t)grp * PK;
    auto count = [&](int pk, int oc) {
        int n = 0;
        if (oc < oc0 + nocl)
            for (int dyi = 0; dyi < kg.ky; ++dyi) {
                const int g = pk * kg.ky + dyi;
                n += off2[g * (c_out + 1) + oc + 1] - off2[g * (c_out + 1) + oc];
            }
        return n;
    };
    // the r-th weight of channel oc in (ic, dx), ordered (dy, dz)
    auto weight = [&](int pk, int oc, int r, int& wd, float& wv) {
        for (int dyi = 0; dyi < kg.ky; ++dyi) {
            const int g = pk * kg.ky + dyi;
            const int lo = off2[g * (c_out + 1) + oc], n = off2[g * (c_out + 1) + oc + 1] - lo;
            if (r < n) {
                const int2 m = meta2[lo + r];
                wd = (oc - oc0) * SLb - ((dyi - kg.hy) * t.ZR + m.y) * (int)sizeof(float);
                wv = val2[lo + r];
                if (!(fabsf(wv) >= 0x1p-50f) && !isnan(wv)) *guard = 1;
                return;
            }
            r -= n;
        }
    };
    int carry = 0;
    for (int p0 = 0; p0 < PK; p0 += blockDim.x) {
        const int pk = p0 + threadIdx.x;
        int tot = 0, full = 0;
        if (pk < PK)
            for (int p = 0; p < npair; ++p) {
                const int na = count(pk, oc0 + 2 * p), nb = count(pk, oc0 + 2 * p + 1);
                tot += max(na, nb);
                full += min(na, nb);
            }
        int all;
        const int ex = block_excl_scan(tot, sm, &all);
        if (pk < PK) {
            const int base = carry + ex;
            PO[pk] = base;
            PF[pk] = full;
            int f = base, sgl = base + full;
            for (int p = 0; p < npair; ++p) {
                const int oa = oc0 + 2 * p, ob = oa + 1;
                const int na = count(pk, oa), nb = count(pk, ob);
                const int m = min(na, nb);
                for (int r = 0; r < m; ++r) {
                    int4 q;
                    float wa, wb;
                    weight(pk, oa, r, q.x, wa);
                    weight(pk, ob, r, q.z, wb);
                    q.y = __float_as_int(wa);
                    q.w = __float_as_int(wb);
                    R[f++] = q;
                }
                const int ol = na > nb ? oa : ob;
                for (int r = m; r < max(na, nb); ++r) {
                    int4 q{0, 0, 0, 0};
                    float wa;
                    weight(pk, ol, r, q.x, wa);
                    q.y = __float_as_int(wa);
                    R[sgl++] = q;
                }
            }
        }
        carry += all;
    }
    if (threadIdx.x == 0) PO[PK] = carry;
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

__device__ __forceinline__ float absent_add(float a, float b, uint32_t marker) {
    if (__float_as_uint(a) == marker) return b;
    if (__float_as_uint(b) == marker) return a;
    return a + b;
}

// warp owning input row i (rows split as A_w = floor(w*nr/8)): floor((8i + 7) / nr), by a float
// reciprocal and one correction each way (8i + 7 < 2^11)
__device__ __forceinline__ int owner_of(int i, int nr, float inv_nr) {
    const int num = 8 * i + 7;
    int q = __float2int_rz((float)num * inv_nr);
    if (q * nr > num) --q;
    if ((q + 1) * nr <= num) ++q;
    return q;
}

// Epilogue rows of one output channel: merge the warps' copies of each row (fixed warp order),
// bias on the support, streaming store of the slice, support count and (with attention) the
// score-digit histogram. Branch-free: lanes off the support increment a private dummy bin past
// the histogram instead of branching around the atomic.
template <int MODE>
__device__ __forceinline__ void epi_rows(const float* S, float* P, float bv, int nyr, int Z, int ZR, int warp,
                                         int lane, uint32_t hist_s, uint32_t& cnt, int yoff, int hy,
                                         uint32_t marker, const uint32_t* rowsrc) {
    const bool vec = (Z & 3) == 0;
    const uint32_t dummy = hist_s + (uint32_t)(kSelBins + lane) * 4u;
    for (int r = warp; r < nyr; r += kFwdWarps) {
        // row yrel = r + yoff (relative to the first input row) has a copy in the region of every
        // warp owning an input row in [yrel - hy, yrel + hy], at region row yrel + hy*(2w + 1)
        const int yrel = r + yoff;
        const uint32_t ow = rowsrc[r];   // source warps of this row (owner table of the tile)
        const int wlo = (int)(ow & 0xffu), whi = (int)(ow >> 8);
        for (int z0 = 4 * lane; z0 < Z; z0 += 128) {
            float v[4];
            {
                const float* A = S + (yrel + hy * (2 * wlo + 1)) * ZR + z0;
                if (vec) {
                    const float4 q = *reinterpret_cast<const float4*>(A);
                    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[e] = z0 + e < Z ? A[e] : __uint_as_float(marker);
                }
            }
            for (int w = wlo + 1; w <= whi; ++w) {   // rows next to a warp boundary: merge copies
                const float* A = S + (yrel + hy * (2 * w + 1)) * ZR + z0;
                float u[4];
                if (vec) {
                    const float4 q = *reinterpret_cast<const float4*>(A);
                    u[0] = q.x; u[1] = q.y; u[2] = q.z; u[3] = q.w;
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) u[e] = z0 + e < Z ? A[e] : __uint_as_float(marker);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) v[e] = absent_add(v[e], u[e], marker);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool pres = __float_as_uint(v[u]) != marker;
                v[u] = pres ? v[u] + bv : __uint_as_float(kAbsent);
                if (MODE == SPC_ATTN_NONE) cnt += pres ? 1u : 0u;   // else: the histogram total
                if (MODE != SPC_ATTN_NONE) {
                    const uint32_t addr = pres ? hist_s + ((score_bits(__float_as_uint(v[u]), MODE) >> 21) << 2) : dummy;
                    asm volatile("red.shared.add.u32 [%0], 1;" :: "r"(addr) : "memory");
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
}

// "add val*fval to buffer at uid" on the shared accumulator; the first update of a voxel
// replaces the absent marker (structural support, reading R3)
// shared-memory load (idle lanes read a harmless in-range word) / predicated store: no branch
// around the read-modify-write
__device__ __forceinline__ float lds_u(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void sts_p(uint32_t addr, float v, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.f32 [%0], %1;\n\t}"
                 :: "r"(addr), "f"(v), "r"((int)p) : "memory");
}

// (-0 mode: the marker is -0.0, which the first fma replaces by the product itself)
template <bool NEG0>
__device__ __forceinline__ float upd(float old, float v, float w) {
    if (NEG0) return fmaf(v, w, old);
    return fmaf(v, w, __float_as_uint(old) == kAbsent ? 0.0f : old);
}

__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

__device__ __forceinline__ int pop_lane(unsigned& m) {
    if (!m) return -1;
    const int j = __ffs(m) - 1;
    m &= m - 1;
    return j;
}

// The accumulate loop of one warp: its input rows of every (ic, input plane) item against the
// item's weight rounds. Each item's first 32 stored inputs stream from global memory into a
// private shared ring with cp.async, kRing - 1 items ahead of the one being processed (no
// block-wide staging); the rare longer runs load their remainder directly. Only the low 32 bits
// of a key are needed: L = key - rowbase < 2^32, so L = key_lo - rowbase_lo (mod 2^32).
template <bool NEG0>
__device__ __forceinline__ void fwd_items(const Geo& gx, const KGeo& kg, const FwdArgs& a, int64_t b, int x,
                                          int A_w, int B_w, int NRP, int ylo, int Z, int ZR, float invZ,
                                          int lane, const uint32_t* rp, const int* pko, const int* pkf,
                                          const int4* rec, unsigned char* ring, const char* accw) {
    const int c_in = (int)gx.C;
    const int PK = c_in * kg.kx;
    const uint32_t accs = (uint32_t)__cvta_generic_to_shared(accw);
    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
    const uint32_t* xk32 = reinterpret_cast<const uint32_t*>(a.xkeys);   // little-endian low words
    for (int pg = 0; pg < PK; pg += 32) {
        // lane j gathers the metadata of item pg + j
        int m_n = 0, m_rb = 0, m_re = 0, m_rf = 0;
        uint32_t m_e0 = 0, m_base = 0;
        if (pg + lane < PK) {
            const int pk = pg + lane;
            const uint32_t* RP = rp + pk * NRP;
            m_e0 = RP[A_w];
            m_n = (int)(RP[B_w] - m_e0);
            m_rb = pko[pk];
            m_re = pko[pk + 1];
            m_rf = m_rb + pkf[pk];
            if (m_rb == m_re) m_n = 0;
            const int ic = pk / kg.kx, xs = x + (pk - ic * kg.kx) - kg.hx;
            m_base = (uint32_t)((uint64_t)(((b * c_in + ic) * gx.X + xs) * (int64_t)gx.Y + ylo) * (uint64_t)Z);
        }
        unsigned iss = __ballot_sync(kFull, m_n > 0), pro = iss;
        auto issue = [&](int jl, int slotk) {
            const uint32_t e = __shfl_sync(kFull, m_e0, jl);
            const int n = __shfl_sync(kFull, m_n, jl);
            if (lane < n) {
                const uint32_t slot = ring_s + (uint32_t)(slotk * kRingSlotB);
                cp_async4(slot + lane * 4u, xk32 + 2 * (size_t)(e + lane));
                cp_async4(slot + 128u + lane * 4u, a.xvals + e + lane);
            }
        };
#pragma unroll
        for (int k = 0; k < kRing - 1; ++k) {   // prologue: kRing - 1 items in flight
            const int jl = pop_lane(iss);
            if (jl >= 0) issue(jl, k);
            cp_async_commit();
        }
        for (int k = 0; pro; ++k) {
            const int jl = pop_lane(pro);
            const int ji = pop_lane(iss);
            if (ji >= 0) issue(ji, (k + kRing - 1) % kRing);   // into the slot freed by item k - 1
            cp_async_commit();
            cp_async_wait<kRing - 1>();   // item k has landed (this lane's copies)
            const int n = __shfl_sync(kFull, m_n, jl);
            const int rb = __shfl_sync(kFull, m_rb, jl), re = __shfl_sync(kFull, m_re, jl);
            const int rf = __shfl_sync(kFull, m_rf, jl);
            const uint32_t rbase = __shfl_sync(kFull, m_base, jl);
            const uint32_t e0 = __shfl_sync(kFull, m_e0, jl);
            const unsigned char* slot = ring + (k % kRing) * kRingSlotB;
            for (int c = 0; c < n; c += 32) {
                const bool valid = c + lane < n;
                int pos = 0;   // idle lanes: position 0 of the warp's region (reads stay in range)
                float v = 0.0f;
                if (valid) {
                    uint32_t klo;
                    if (c == 0) {
                        klo = reinterpret_cast<const uint32_t*>(slot)[lane];
                        v = reinterpret_cast<const float*>(slot + 128)[lane];
                    } else {   // remainder of a long run: direct loads
                        const uint32_t e = e0 + (uint32_t)(c + lane);
                        klo = xk32[2 * (size_t)e];
                        v = a.xvals[e];
                    }
                    const uint32_t L = klo - rbase;
                    const uint32_t yrel = div_small(L, (uint32_t)Z, invZ);
                    pos = (int)(yrel * (uint32_t)ZR + (L - yrel * (uint32_t)Z));
                }
                const uint32_t base = accs + (uint32_t)pos * 4u;
                // two-channel rounds: both read-modify-writes in flight (distinct slices);
                // predicated shared loads/stores (no branch), the next round's record prefetched
                int4 q = rec[rb];
#pragma unroll 2
                for (int r = rb; r < rf; ++r) {
                    const int4 qn = rec[r + 1];   // rec[re] stays inside shared memory (pko follows)
                    const uint32_t pa = base + (uint32_t)q.x, pb = base + (uint32_t)q.z;
                    const float oa = lds_u(pa), ob = lds_u(pb);
                    sts_p(pa, upd<NEG0>(oa, v, __int_as_float(q.y)), valid);
                    sts_p(pb, upd<NEG0>(ob, v, __int_as_float(q.w)), valid);
                    __syncwarp();   // the next round's lanes may read what this one wrote
                    q = qn;
                }
#pragma unroll 1
                for (int r = rf; r < re; ++r) {
                    const int4 qn = rec[r + 1];
                    const uint32_t pa = base + (uint32_t)q.x;
                    sts_p(pa, upd<NEG0>(lds_u(pa), v, __int_as_float(q.y)), valid);
                    q = qn;
                    __syncwarp();
                }
            }
        }
        cp_async_wait<0>();
        __syncwarp();
    }
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
    const int SL = t.RT * ZR;                        // floats per output-channel slice

    // shared layout (float offsets, 16-byte aligned pieces):
    // [pad][acc ocg*RT*ZR][pad] | misc(512) | rounds | pko | pkf | rp | cp.async rings (= hist in the epilogue)
    const int PK = c_in * kg.kx;                     // (ic, input plane) work items
    const int ylo = max(0, y0 - kg.hy), yhi = min(gy.Y, ye + kg.hy);
    const int nr = yhi - ylo;                        // input rows read per plane
    const int NRP = nr + 1;
    float* acc = smf + t.pad;
    uint32_t* misc = reinterpret_cast<uint32_t*>(smf + 2 * t.pad + t.ocg * SL);
    int4* rec = reinterpret_cast<int4*>(misc + 512);   // misc: scan scratch [0, 64), row owners [64, 64 + TY)
    int* pko = reinterpret_cast<int*>(rec + t.nwg_max);
    int* pkf = pko + ((PK + 1 + 3) & ~3);
    uint32_t* rp = reinterpret_cast<uint32_t*>(pkf + ((PK + 1 + 3) & ~3));
    unsigned char* ring = reinterpret_cast<unsigned char*>(rp + ((PK * (t.TY + 2 * kg.hy + 1) + 3) & ~3));
    uint32_t* hist = reinterpret_cast<uint32_t*>(ring);   // epilogue only

    const bool neg0 = *a.guard == 0;                 // -0 accumulation mode (value_guard_kernel)
    const uint32_t marker = neg0 ? kNegZero : kAbsent;
    {
        const int n4 = (2 * t.pad + t.ocg * SL) / 4;
        uint4 ab = make_uint4(marker, marker, marker, marker);
        for (int i = threadIdx.x; i < n4; i += blockDim.x) reinterpret_cast<uint4*>(smf)[i] = ab;
    }
    const int* gpko = a.pkoff + (int64_t)blockIdx.y * (PK + 1);
    for (int i = threadIdx.x; i <= PK; i += blockDim.x) pko[i] = gpko[i];
    for (int i = threadIdx.x; i < PK; i += blockDim.x) pkf[i] = a.pkfull[(int64_t)blockIdx.y * PK + i];

    // Warp w owns input rows [A_w, B_w) (relative to ylo) and writes into a private region of the
    // accumulator: input row yrel lands at region row yrel + hy*(2w + 1), so targets (rows
    // yrel - oy, |oy| <= hy) of different warps never meet; the epilogue merges the copies.
    const int A_w = (warp * nr) / kFwdWarps, B_w = ((warp + 1) * nr) / kFwdWarps;
    const int cw = kg.hy * (2 * warp + 1) * ZR;
    const float invZ = 1.0f / (float)Z;
    // row pointers of every (ic, input plane), rows ylo..yhi, in one burst
    for (int q = threadIdx.x; q < PK * NRP; q += blockDim.x) {
        const int pk = q / NRP, r = q - pk * NRP;
        const int ic = pk / kg.kx, pl = pk - ic * kg.kx;
        const int xs = x + pl - kg.hx;
        rp[q] = (xs >= 0 && xs < gx.X) ? a.xrow[((b * c_in + ic) * gx.X + xs) * (int64_t)gx.Y + ylo + r] : 0u;
    }
    {   // this group's weight rounds (fwd_rounds_kernel), one coalesced copy
        const int4* grec = a.rec + (int64_t)blockIdx.y * t.nwg_max;
        const int nrec = gpko[PK];
        for (int i = threadIdx.x; i < nrec; i += blockDim.x) rec[i] = grec[i];
    }
    __syncthreads();   // row pointers, tables and rounds in shared memory
    // ------------------------------------------------------------ accumulate (Alg. 1 inner loops)
    if (A_w < B_w) {
        const char* accw = reinterpret_cast<const char*>(acc + cw);
        unsigned char* ring_w = ring + warp * (kRing * kRingSlotB);
        if (neg0)
            fwd_items<true>(gx, kg, a, b, x, A_w, B_w, NRP, ylo, Z, ZR, invZ, lane, rp, pko, pkf, rec, ring_w, accw);
        else
            fwd_items<false>(gx, kg, a, b, x, A_w, B_w, NRP, ylo, Z, ZR, invZ, lane, rp, pko, pkf, rec, ring_w, accw);
    }
    __syncthreads();   // accumulator complete; rings free for the histogram

    // ------------------------------------------------------------------------ epilogue
    // "get non-zero entries" and "add bias to non-zero entries": the tile's slice
    // of the pre-attention responses goes to the (b, oc) buffers -- the paper's temporary dense
    // buffer, absent marker where there is no support -- while the support size and a
    // histogram of the top score digit are accumulated for the attention threshold.
    const int nyr = ye - y0;
    const bool do_hist = a.attn != SPC_ATTN_NONE;
    // output row r has copies in the regions of the warps owning input rows yrel-hy..yrel+hy
    uint32_t* rowsrc = misc + 64;
    {
        const float inv_nr = 1.0f / (float)nr;
        for (int r = threadIdx.x; r < nyr; r += blockDim.x) {
            const int yrel = r + (y0 - ylo);
            const int wlo = owner_of(max(0, yrel - kg.hy), nr, inv_nr), whi = owner_of(min(nr - 1, yrel + kg.hy), nr, inv_nr);
            rowsrc[r] = (uint32_t)wlo | ((uint32_t)whi << 8);
        }
    }
    const uint32_t hist_s = (uint32_t)__cvta_generic_to_shared(hist);
    for (int ocl = 0; ocl < nocl; ++ocl) {
        const int oc = oc0 + ocl;
        const int64_t s = b * c_out + oc;
        const float bv = a.bias ? a.bias[oc] : 0.0f;
        const float* S = acc + ocl * SL;
        if (do_hist)
            for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        uint32_t cnt = 0;
        float* P = a.pre + s * gy.V + ((int64_t)x * gy.Y + y0) * Z;
        const int yoff = y0 - ylo;
        if (a.attn == SPC_ATTN_MAGNITUDE)
            epi_rows<SPC_ATTN_MAGNITUDE>(S, P, bv, nyr, Z, ZR, warp, lane, hist_s, cnt, yoff, kg.hy, marker, rowsrc);
        else if (a.attn == SPC_ATTN_RAW)
            epi_rows<SPC_ATTN_RAW>(S, P, bv, nyr, Z, ZR, warp, lane, hist_s, cnt, yoff, kg.hy, marker, rowsrc);
        else
            epi_rows<SPC_ATTN_NONE>(S, P, bv, nyr, Z, ZR, warp, lane, hist_s, cnt, yoff, kg.hy, marker, rowsrc);
        if (do_hist) {   // merge the tile histogram; support size = its total
            __syncthreads();
            for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) {
                const uint32_t h = hist[i];
                cnt += h;
                if (h) atomicAdd(&a.hist[s * kSelBins + i], h);
            }
        }
        const uint32_t tot = block_sum(cnt, misc);
        if (threadIdx.x == 0 && tot) atomicAdd(&a.seg_count[s], (unsigned long long)tot);
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
            a.stg_cnt[s] = (uint64_t)n;
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
                a.stg_cnt[s] = cum + h[bin];   // digits >= B1
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
template <int MODE>
__device__ __forceinline__ void classify_chunk(const FwdArgs& a, const FwdSeg& st, int64_t s, int64_t c, int64_t V,
                                               const uint32_t (&bits)[kChunkItems], int64_t lo,
                                               unsigned long long* sm, uint2* sbuf) {
    // digit of each value, -1 off the support: kept outright iff d > B1, candidate iff d == B1;
    // staged iff d >= B1 (the write pass then never touches the dense buffer again)
    uint32_t ge = 0, cand = 0;
#pragma unroll
    for (int u = 0; u < kChunkItems; ++u) {
        const bool pres = bits[u] != kAbsent;
        // keep-all: every support entry is "definite" (digit forced above B1)
        const int dig = st.keep_all ? (int)st.b1 + 1 : (int)(score_bits(bits[u], MODE) >> 21);
        const int d = pres ? dig : -1;
        ge |= (uint32_t)(d >= (int)st.b1) << u;
        cand += (uint32_t)(d == (int)st.b1);
    }
    // one scan of 4 x 12-bit per-slab staged counts | 16-bit candidate count: key-ordered slots
    unsigned long long packed = (unsigned long long)cand << 48;
#pragma unroll
    for (int v = 0; v < 4; ++v) packed |= (unsigned long long)__popc((ge >> (4 * v)) & 15u) << (12 * v);
    unsigned long long tot;
    const unsigned long long ex = block_excl_scan(packed, sm, &tot);
    uint32_t nge = 0;
#pragma unroll
    for (int v = 0; v < 4; ++v) nge += (uint32_t)((tot >> (12 * v)) & 0xfffu);
    const uint32_t tcand = (uint32_t)(tot >> 48);
    __shared__ uint64_t sh_base, sh_cbase;
    __shared__ uint32_t sh_ccur;
    const int64_t it = s * a.nchunk + c;
    if (threadIdx.x == 0) {
        a.tile_def[it] = nge - tcand;
        a.chunk_ge[it] = nge;
        const uint64_t b0 = nge ? a.stg_off[s] + atomicAdd(&a.stg_cur[s], (unsigned long long)nge) : 0ull;
        a.chunk_stg[it] = b0;
        sh_base = b0;
        sh_cbase = tcand ? a.cand_off[s] + atomicAdd(&a.cand_cur[s], (unsigned long long)tcand) : 0ull;
        sh_ccur = 0;
    }
    if (nge == 0) return;   // block-uniform
    // stage this thread's entries at their key-ordered slots (predicated shared stores)
    uint32_t slab0 = 0;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        uint32_t q = slab0 + (uint32_t)((ex >> (12 * v)) & 0xfffu);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int u = 4 * v + w;
            const bool k = (ge >> u) & 1u;
            const uint32_t p = (uint32_t)lo + 4u * ((uint32_t)v * kChunkThreads + threadIdx.x) + (uint32_t)w;
            if (k) sbuf[q] = make_uint2(p, bits[u]);
            q += k ? 1u : 0u;
        }
        slab0 += (uint32_t)((tot >> (12 * v)) & 0xfffu);
    }
    __syncthreads();
    // coalesced copy to the staging list; candidates (digit == B1) also appended, any order
    uint2* out = a.stg + sh_base;
    const int lane = threadIdx.x & 31;
    for (uint32_t i0 = threadIdx.x & ~31u; i0 < nge; i0 += kChunkThreads) {
        const uint32_t i = i0 + lane;
        const bool ok = i < nge;
        const uint2 e = ok ? sbuf[i] : make_uint2(0u, kAbsent);
        if (ok) out[i] = e;
        const bool is_c = ok && !st.keep_all && (score_bits(e.y, MODE) >> 21) == st.b1;
        const unsigned m = __ballot_sync(kFull, is_c);
        if (m) {
            uint32_t slot = 0;
            if (lane == 0) slot = atomicAdd(&sh_ccur, (uint32_t)__popc(m));
            slot = __shfl_sync(kFull, slot, 0);
            if (is_c) a.cand[sh_cbase + slot + __popc(m & ((1u << lane) - 1u))] = e;
        }
    }
}

__global__ void __launch_bounds__(kChunkThreads) fwd_classify_kernel(FwdArgs a, int64_t V) {
    const int64_t s = blockIdx.x / a.nchunk, c = blockIdx.x % a.nchunk;
    const FwdSeg st = a.seg[s];
    const int64_t lo = c * kChunk;
    const float* P = a.pre + s * V;
    __shared__ unsigned long long sm[33];
    __shared__ uint2 sbuf[kChunk];   // the chunk's candidates, staged for a coalesced write
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
    if (a.attn == SPC_ATTN_RAW) classify_chunk<SPC_ATTN_RAW>(a, st, s, c, V, bits, lo, sm, sbuf);
    else classify_chunk<SPC_ATTN_MAGNITUDE>(a, st, s, c, V, bits, lo, sm, sbuf);   // NONE: keep_all
}

// resolve: the `need` largest composite keys among the candidates of a segment -> kstar; then
// count selected candidates per chunk. All candidates share the top 11 bits (digit B1), so the
// radix select starts below them: an 11-bit digit over the candidate list in HBM, after which
// the survivors (about n/2048) are copied to shared memory and the remaining digits (8, 8, 8,
// 8, 8, 2 bits) run there. All composite keys are distinct (p is unique), so kstar is exact.
constexpr int kResThreads = 512;
constexpr int kResCap = 2048;   // survivors kept in shared memory
__global__ void __launch_bounds__(kResThreads) fwd_resolve_kernel(FwdArgs a) {
    const int64_t s = blockIdx.x;
    FwdSeg st = a.seg[s];
    if (st.keep_all) return;
    const uint64_t n = a.cand_cnt[s];
    const uint2* c = a.cand + a.cand_off[s];
    __shared__ uint32_t h[kSelBins];
    __shared__ uint64_t sc[kResCap];
    __shared__ uint64_t sh_prefix, sh_mask;
    __shared__ int64_t sh_need;
    __shared__ uint32_t sh_bin_cnt, sh_ns;
    if (threadIdx.x == 0) {
        sh_prefix = (uint64_t)st.b1 << 53;
        sh_mask = (uint64_t)(kSelBins - 1) << 53;
        sh_need = st.need;
        sh_ns = 0;
    }
    bool in_smem = false;
    uint32_t ns = 0;
#pragma unroll 1
    for (int pass = 0; pass < 7; ++pass) {
        const int sh = pass < 6 ? 42 - 8 * pass : 0;            // bits 52..42, 41..34, ..., 9..2, 1..0
        const int nb = pass == 0 ? kSelBins : (pass < 6 ? 256 : 4);
        for (int i = threadIdx.x; i < nb; i += blockDim.x) h[i] = 0;
        __syncthreads();
        const uint64_t prefix = sh_prefix, mask = sh_mask;
        const uint32_t dmask = (uint32_t)nb - 1u;
        if (!in_smem) {
            for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
                const uint2 e = c[i];
                const uint64_t k = composite(score_bits(e.y, a.attn), e.x);
                if ((k & mask) == prefix) atomicAdd(&h[(uint32_t)(k >> sh) & dmask], 1u);
            }
        } else {
            for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) {
                const uint64_t k = sc[i];
                if ((k & mask) == prefix) atomicAdd(&h[(uint32_t)(k >> sh) & dmask], 1u);
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            // warp scan of the bins from the top: lane l owns bins nb-1-per*l .. nb-per*(l+1)
            const int l = threadIdx.x, per = nb >= 32 ? nb / 32 : 1;
            uint32_t own = 0;
            if (l * per < nb)
                for (int q = 0; q < per; ++q) own += h[nb - 1 - per * l - q];
            const uint32_t incl = warp_incl_scan(own);
            const int64_t need = sh_need;
            const int64_t before = (int64_t)(incl - own);
            if (own && before < need && before + (int64_t)own >= need) {
                int64_t cum = before;
                for (int q = 0; q < per; ++q) {
                    const int bin = nb - 1 - per * l - q;
                    if (cum + (int64_t)h[bin] >= need) {
                        sh_need = need - cum;
                        sh_prefix = prefix | ((uint64_t)bin << sh);
                        sh_mask = mask | ((uint64_t)dmask << sh);
                        sh_bin_cnt = h[bin];
                        break;
                    }
                    cum += h[bin];
                }
            }
        }
        __syncthreads();
        if (!in_smem && pass + 1 < 7 && sh_bin_cnt <= (uint32_t)kResCap) {
            // survivors of the chosen prefix -> shared memory (order irrelevant: keys distinct)
            const uint64_t p2 = sh_prefix, m2 = sh_mask;
            for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) {
                const uint2 e = c[i];
                const uint64_t k = composite(score_bits(e.y, a.attn), e.x);
                if ((k & m2) == p2) sc[atomicAdd(&sh_ns, 1u)] = k;
            }
            __syncthreads();
            ns = sh_ns;
            in_smem = true;
        }
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

// Elements are loaded as in classify (slab v = 0..3 of 256 float4, thread t holds voxels
// lo + 4*(v*256 + t) + w): coalesced. Key order within the chunk is (v, t, w), so one scan of
// four packed 16-bit per-slab counts gives every thread the output slot of each of its slabs.
// write: keep iff composite(score, p) >= kstar (every staged entry when keep-all); ordered
// compaction in key order ("compress ids ... write k largest features"). One warp per
// chunk over its staged run (entries with digit >= B1, already in key order).
constexpr int kWriteWarps = 8;
__global__ void __launch_bounds__(32 * kWriteWarps) fwd_write_kernel(FwdArgs a, int64_t V) {
    const int lane = threadIdx.x & 31;
    const int64_t it = (int64_t)blockIdx.x * kWriteWarps + (threadIdx.x >> 5);
    if (it >= a.nseg * a.nchunk) return;
    const int64_t s = it / a.nchunk;
    const FwdSeg st = a.seg[s];
    const uint32_t n = a.chunk_ge[it];
    if (n == 0) return;
    const uint2* in = a.stg + a.chunk_stg[it];
    uint64_t out = a.seg_off[s] + a.tile_off[it];
    const uint64_t kb = (uint64_t)s * (uint64_t)V;
    // composite(score, p) = (score << 32 | ~p) >= kstar, as two 32-bit compares
    const uint32_t ks = (uint32_t)(st.kstar >> 32), kp = (uint32_t)st.kstar;
    for (uint32_t i0 = 0; i0 < n; i0 += 32) {
        const uint32_t i = i0 + lane;
        const bool ok = i < n;
        const uint2 e = ok ? in[i] : make_uint2(0u, kAbsent);
        const uint32_t sc = score_bits(e.y, a.attn);
        const bool keep = ok && (st.keep_all || sc > ks || (sc == ks && ~e.x >= kp));
        const unsigned m = __ballot_sync(kFull, keep);
        if (keep) {
            const uint64_t q = out + __popc(m & ((1u << lane) - 1u));
            a.out_keys[q] = kb + e.x;
            a.out_vals[q] = __uint_as_float(e.y);
        }
        out += __popc(m);
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
    cudaMemsetAsync(a.stg_cur, 0, segb, s);
    cudaMemsetAsync(a.tile_sel, 0, sizeof(uint32_t) * (size_t)(nseg * a.nchunk), s);
    if (a.attn != SPC_ATTN_NONE) cudaMemsetAsync(a.hist, 0, sizeof(uint32_t) * kSelBins * (size_t)nseg, s);
    const dim3 grid((unsigned)(gy.B * gy.X * t.nty), (unsigned)t.n_ocg);
    const unsigned sgrid = (unsigned)(nseg * a.nchunk);
    cudaMemsetAsync(a.guard, 0, sizeof(int), s);
    {
        SPC_PHASE("value_guard", s, 1);
        value_guard_kernel<<<148 * 4, 256, 0, s>>>(a.xvals, a.x_nnz_dev, a.x_nnz, a.guard);
    }
    {
        SPC_PHASE("fwd_rounds", s, 1);
        fwd_rounds_kernel<<<(unsigned)t.n_ocg, 128, 0, s>>>(kg, (int)gx.C, (int)gy.C, t, a.meta2, a.val2, a.off2,
                                                          a.rec, a.pkoff, a.pkfull, a.guard);
    }
    { SPC_PHASE("conv_fwd", s, 1); conv_fwd_kernel<<<grid, kFwdThreads, t.smem, s>>>(gx, gy, kg, t, a); }
    { SPC_PHASE("fwd_find", s, 1); fwd_find_kernel<<<(unsigned)nseg, 256, 0, s>>>(a, nseg); }
    {
        SPC_PHASE("seg_scan", s, a.attn != SPC_ATTN_NONE ? 2 : 1);
        if (a.attn != SPC_ATTN_NONE) seg_scan_u64_kernel<<<1, 1024, 0, s>>>(a.cand_cnt, a.cand_off, nseg, nullptr);
        seg_scan_u64_kernel<<<1, 1024, 0, s>>>(a.stg_cnt, a.stg_off, nseg, nullptr);
    }
    { SPC_PHASE("fwd_classify", s, 1); fwd_classify_kernel<<<sgrid, kChunkThreads, 0, s>>>(a, gy.V); }
    if (a.attn != SPC_ATTN_NONE) {
        SPC_PHASE("fwd_resolve", s, 1);
        fwd_resolve_kernel<<<(unsigned)nseg, kResThreads, 0, s>>>(a);
    }
    // kept per segment goes to cand_cnt (reused as scratch), then segment offsets
    { SPC_PHASE("fwd_chunk_scan", s, 1); fwd_chunk_scan_kernel<<<(unsigned)nseg, 256, 0, s>>>(a, a.cand_cnt); }
    { SPC_PHASE("seg_scan", s, 1); seg_scan_u64_kernel<<<1, 1024, 0, s>>>(a.cand_cnt, a.seg_off, nseg, a.out_nnz); }
    { SPC_PHASE("fwd_write", s, 1); fwd_write_kernel<<<(unsigned)((nseg * a.nchunk + kWriteWarps - 1) / kWriteWarps), 32 * kWriteWarps, 0, s>>>(a, gy.V); }
    return cudaGetLastError();
}

}  // namespace spc

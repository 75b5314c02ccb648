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
#include <cstdlib>
#ifdef SPC_DEBUG
#include <cstdio>
#endif

namespace spc {

constexpr int kFwdThreads = 256;
constexpr int kFwdWarps = kFwdThreads / 32;   // warp w accumulates output channel oc0 + w
constexpr size_t kFwdBudget = 113 * 1024;     // two CTAs (16 warps) per SM
constexpr size_t kFwdBudgetMax = 220 * 1024;  // one CTA per SM (very long rows)
constexpr int kStageCap = 1536;               // staged input entries per chunk (byte position + value)
static_assert(kStageCap * 8 >= (kSelBins + 32) * 4, "the epilogue histogram (+ 32 dummy bins) reuses the staging area");

__host__ __device__ inline size_t r4(size_t n) { return (n + 3) & ~(size_t)3; }

// shared-memory bytes beyond the accumulator: staging, item tables (flat offset, first global
// entry, row base), round offsets and round records of the group, scratch
static size_t fwd_fixed_smem(int PK, int ocg, int64_t nwg) {
    return (size_t)kStageCap * 8 + 4 * (4 * r4(PK + 1) + r4(kStageCap / 64 + PK + 1) + 80) +
           8 * ((size_t)ocg * PK + (size_t)nwg + 1) + 64;
}

FwdTile plan_fwd_tile(const Geo& gy, const KGeo& kg, int c_out, int c_in, int64_t nw_total, double rho_in) {
    FwdTile t{};
    const int cz = ((kg.hz + 3) / 4) * 4;                         // column of z = 0 (16-byte aligned rows)
    const int ZR = (int)r4((size_t)cz + gy.Z + kg.hz);
    const int PK = c_in * kg.kw * kg.kx;   // items (ic, input plane offset (dw, dx))
    auto nwg = [&](int ocg) { return std::min<int64_t>(nw_total, (int64_t)ocg * c_in * kg.KV); };
    // round records live in shared memory when small; large filter banks (e.g. 32 x 32 x 27) are
    // read through L1 instead of being copied into every CTA
    auto rec_sm = [&](int ocg) { return nwg(ocg) * 8 <= 16 * 1024; };
    // accumulator rows per channel: the band plus 2hy margin rows on each side that catch the
    // updates leaving the band (margin mode), or only the band with those updates predicated off
    // (pred mode: taller bands in the same shared memory, one compare per update)
    auto need = [&](int ocg, int TY, bool pred) {
        // (records in global memory: a 32-record buffer per warp for the current descriptor's)
        return fwd_fixed_smem(PK, ocg, rec_sm(ocg) ? nwg(ocg) : kFwdWarps * 32) +
               (size_t)ocg * (TY + (pred ? 0 : 4 * kg.hy)) * ZR * sizeof(float);
    };
    if (PK >= (1 << 13)) { t.smem = 0; return t; }                 // work descriptors hold 13-bit items
    size_t kFwdBudget = spc::kFwdBudget;
    if (const char* e = getenv("SPC_FWD_BUDGET_KB")) kFwdBudget = (size_t)atoi(e) * 1024;
    int ocg = std::min(c_out, kFwdWarps);
    while (ocg > 1 && need(ocg, 1, true) > kFwdBudget) --ocg;
    // rows too long for two CTAs per SM (a band row of one channel above ~25 k columns): one CTA
    // per SM with the whole shared memory (1D signals up to ~50 k columns)
    if (need(ocg, 1, true) > kFwdBudget) kFwdBudget = kFwdBudgetMax;
    if (need(ocg, 1, true) > kFwdBudget) { t.smem = 0; return t; }
    auto tymax = [&](bool pred) {
        int v = 0;
        while (v < gy.Y && need(ocg, v + 1, pred) <= kFwdBudget) ++v;
        return v;
    };
    // pred mode only when it saves bands and the input is sparse (measured: C4 at 2 % 4.33 ->
    // 4.28 ms, 7 bands instead of 8; at 5 % the per-update compare costs more than the band
    // saves, 14.4 -> 14.9 ms per step; the C3 32 -> 64 layer keeps 2 bands either way and runs
    // 7 % slower predicated). rho_in: input density (upper bound when the count is on the device)
    const int tm = tymax(false), tp = tymax(true);
    bool pred = tm < 1 || ((gy.Y + tp - 1) / tp < (gy.Y + tm - 1) / tm && rho_in <= 0.03);
    if (const char* e = getenv("SPC_FWD_PRED")) pred = e[0] == '1' || tm < 1;
    int TYmax = pred ? tp : tm;
    if (const char* e = getenv("SPC_FWD_TY")) TYmax = std::max(1, std::min(TYmax, atoi(e)));
    const int nty = (gy.Y + TYmax - 1) / TYmax;
    t.TY = (gy.Y + nty - 1) / nty;                                   // balanced bands
    t.nty = nty;
    t.ocg = ocg;
    t.n_ocg = (c_out + ocg - 1) / ocg;
    t.ZR = ZR;
    t.cz = cz;
    t.pred = pred ? 1 : 0;
    t.RA = t.TY + (pred ? 0 : 4 * kg.hy);
    t.PK = PK;
    t.nwg_max = (int)nwg(ocg);
    t.rec_smem = rec_sm(ocg) ? 1 : 0;
    t.smem = need(ocg, t.TY, pred);
    t.fd_nty = make_fastdiv((uint32_t)t.nty);
    t.fd_X = make_fastdiv((uint32_t)gy.X);
    t.fd_Z = make_fastdiv((uint32_t)gy.Z);
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
// fval} in filter(oc, ic)"; here the stored weights of (oc, ic, input plane dx) form the
// rounds of work item (ic, dx) for the warp of oc, ordered (dy, dz). Round record {wd, w}: wd =
// byte offset from an input's accumulator position to its target uid = id - (fid - centre)
// = -(dy - hy) rows - (dz - hz) columns, plus the channel slice of oc.
__global__ void fwd_rounds_kernel(KGeo kg, int c_in, int c_out, FwdTile t, const int2* __restrict__ meta2,
                                  const float* __restrict__ val2, const int* __restrict__ off2, int2* __restrict__ rnd,
                                  int* __restrict__ roff, int* __restrict__ guard) {
    __shared__ int sm[33];
    const int grp = blockIdx.x, oc0 = grp * t.ocg, nocl = min(t.ocg, c_out - oc0);
    const int PK = t.PK, NQ = t.ocg * PK;
    const int SLb = t.RA * t.ZR * (int)sizeof(float);
    int2* R = rnd + (int64_t)grp * t.nwg_max;
    int* RO = roff + (int64_t)grp * (NQ + 1);
    int carry = 0;
    for (int q0 = 0; q0 < NQ; q0 += blockDim.x) {
        const int q = q0 + threadIdx.x;            // q = ocl*PK + pk
        const int ocl = q / PK, pk = q - (q / PK) * PK;
        const int KWX = kg.kw * kg.kx;                 // plane offsets (dw, dx) per input channel
        const int ic = pk / KWX, dx = pk - (pk / KWX) * KWX;
        const int oc = oc0 + ocl;
        int n = 0;
        if (q < NQ && ocl < nocl)
            for (int dy = 0; dy < kg.ky; ++dy) {
                const int g = (ic * KWX + dx) * kg.ky + dy;
                n += off2[g * (c_out + 1) + oc + 1] - off2[g * (c_out + 1) + oc];
            }
        int all;
        const int ex = block_excl_scan(n, sm, &all);
        if (q < NQ) {
            int f = carry + ex;
            RO[q] = f;
            if (ocl < nocl)
                for (int dy = 0; dy < kg.ky; ++dy) {
                    const int g = (ic * KWX + dx) * kg.ky + dy;
                    const int lo = off2[g * (c_out + 1) + oc], hi = off2[g * (c_out + 1) + oc + 1];
                    for (int j = lo; j < hi; ++j) {
                        const float wv = val2[j];
                        if (!(fabsf(wv) >= 0x1p-50f) && !isnan(wv)) *guard = 1;
                        const int wd = ocl * SLb - ((dy - kg.hy) * t.ZR + meta2[j].y) * (int)sizeof(float);
                        R[f++] = make_int2(wd, __float_as_int(wv));
                    }
                }
        }
        carry += all;
    }
    if (threadIdx.x == 0) RO[NQ] = carry;
}

__device__ __forceinline__ uint64_t composite(uint32_t sc, uint32_t p) {
    return ((uint64_t)sc << 32) | (uint64_t)(0xffffffffu - p);
}

// Sampled-pass epilogue rows of one output channel: bias on the support, support count and
// the score-digit histogram (the responses themselves are not stored). Branch-free: lanes off
// the support increment a private dummy bin past the histogram instead of branching around the
// atomic.
template <int MODE>
__device__ __forceinline__ void epi_hist_rows(const float* S, float bv, int nyr, int Z, int ZR, uint32_t hist_s,
                                              uint32_t marker) {
    const bool vec = (Z & 3) == 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t dummy = hist_s + (uint32_t)(kSelBins + lane) * 4u;
    for (int r = warp; r < nyr; r += kFwdWarps) {
        for (int z0 = 4 * lane; z0 < Z; z0 += 128) {
            const float* A = S + r * ZR + z0;
            float v[4];
            if (vec) {
                const float4 q = *reinterpret_cast<const float4*>(A);
                v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) v[e] = z0 + e < Z ? A[e] : __uint_as_float(marker);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool pres = __float_as_uint(v[u]) != marker;
                const uint32_t addr =
                    pres ? hist_s + ((score_bits(__float_as_uint(v[u] + bv), MODE) >> 21) << 2) : dummy;
                asm volatile("red.shared.add.u32 [%0], 1;" :: "r"(addr) : "memory");
            }
        }
    }
}

// Candidate epilogue of one output channel (warp = channel, no block barrier): "get non-zero
// entries" (structural support R3), "add bias", and every support entry whose score
// reaches the segment's threshold tlow is appended in key order to the tile's candidate run.
// Row by row, 128 voxels per step: lane l holds z = z0 + l + 32u (u = 0..3), so each of the four
// 32-voxel groups is one ballot. Candidates are ranked into a per-warp shared-memory buffer
// as (position, value) pairs -- one 8-byte store per candidate, none for the other lanes, so a
// 32-voxel group costs one shared-memory wavefront when it has candidates -- and the buffer is
// flushed to the run with coalesced stores. Returns the run length and the largest candidate
// score.
constexpr int kCandBuf = 192;   // per-warp buffer entries, in the staging area
template <int MODE, bool FULL>   // FULL: Z is a multiple of 128 (no ragged 128-voxel slot)
__device__ __forceinline__ void epi_cand(const float* S, int nyr, int Z, int ZR, float bv, uint32_t tlow,
                                         uint32_t marker, uint32_t pbase, uint32_t* __restrict__ cpos,
                                         float* __restrict__ cval, uint2* buf, uint32_t& n_out, uint32_t& max_out) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t bufs = (uint32_t)__cvta_generic_to_shared(buf);
    uint32_t nb = 0, nf = 0, mx = 0;   // buffered, flushed
    // 128-voxel slots in key order (row, z0); two slots per step, their eight loads issued first
    const int nz0 = (Z + 127) >> 7, nslot = nyr * nz0;
    int r_s = 0, zi_s = 0;   // (row, 128-voxel column) of slot s0, advanced without divisions
    for (int s0 = 0; s0 < nslot; s0 += 2) {
        float raw[8];
        uint32_t pz[8];
        int r = r_s, zi = zi_s;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int sl = s0 + h;
            const int z0 = zi << 7;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int z = z0 + 32 * u + lane;
                const bool in = sl < nslot && (FULL || z < Z);
                raw[4 * h + u] = in ? S[r * ZR + z] : __uint_as_float(marker);
                pz[4 * h + u] = pbase + (uint32_t)(r * Z + z);
            }
            if (++zi == nz0) { zi = 0; ++r; }
        }
        r_s = r;
        zi_s = zi;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = 4 * h + u;
                const bool pres = __float_as_uint(raw[q]) != marker;
                const float val = raw[q] + bv;
                const uint32_t sc = MODE == SPC_ATTN_NONE ? 0u : score_bits(__float_as_uint(val), MODE);
                const bool c = pres && sc >= tlow;
                mx = c ? max(mx, sc) : mx;
                const uint32_t bal = __ballot_sync(kFull, c);
                {   // predicated 8-byte store (no branch): only candidate lanes write
                    const uint32_t ad = bufs + 8u * (nb + (uint32_t)__popc(bal & lt));
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t@p st.shared.v2.u32 [%0], {%1, %2};\n\t}"
                                 :: "r"(ad), "r"(pz[q]), "r"(__float_as_uint(val)), "r"((int)c) : "memory");
                }
                nb += (uint32_t)__popc(bal);
            }
            if (nb > kCandBuf - 128) {   // flush: coalesced copy of the buffer to the run
                __syncwarp();
                for (uint32_t i = lane; i < nb; i += 32) {
                    const uint2 e = buf[i];
                    cpos[nf + i] = e.x;
                    cval[nf + i] = __uint_as_float(e.y);
                }
                nf += nb;
                nb = 0;
                __syncwarp();
            }
        }
    }
    __syncwarp();
    for (uint32_t i = lane; i < nb; i += 32) {
        const uint2 e = buf[i];
        cpos[nf + i] = e.x;
        cval[nf + i] = __uint_as_float(e.y);
    }
    n_out = nf + nb;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, d));
    max_out = mx;
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
// predicated load: idle lanes do not touch shared memory (no benign read/write overlap with an
// active lane's target, so racecheck stays silent)
__device__ __forceinline__ float lds_p(uint32_t addr, bool p) {
    float v = 0.0f;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.shared.f32 %0, [%1];\n\t}"
                 : "+f"(v) : "r"(addr), "r"((int)p) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" :: "r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void sts_p(uint32_t addr, float v, bool p) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.f32 [%0], %1;\n\t}"
                 :: "r"(addr), "f"(v), "r"((int)p) : "memory");
}

// -0 mode RMW of the lane's two entries in one predicated block: loads, fmas and stores under
// the entries' predicates, no zero-initialised temporaries (the same instructions the C++ form
// needs, minus the moves and selects the compiler adds around conditional asm outputs)
__device__ __forceinline__ void rmw2_neg0(uint32_t qa, uint32_t qb, float va, float vb, float w, int oka, int okb) {
    asm volatile(
        "{\n\t.reg .pred pa, pb;\n\t.reg .f32 ta, tb;\n\t"
        "setp.ne.b32 pa, %5, 0;\n\tsetp.ne.b32 pb, %6, 0;\n\t"
        "@pa ld.shared.f32 ta, [%0];\n\t@pb ld.shared.f32 tb, [%1];\n\t"
        "@pa fma.rn.f32 ta, %2, %4, ta;\n\t@pb fma.rn.f32 tb, %3, %4, tb;\n\t"
        "@pa st.shared.f32 [%0], ta;\n\t@pb st.shared.f32 [%1], tb;\n\t}"
        :: "r"(qa), "r"(qb), "f"(va), "f"(vb), "f"(w), "r"(oka), "r"(okb) : "memory");
}
__device__ __forceinline__ void rmw1_neg0(uint32_t qa, float va, float w, int oka) {
    asm volatile(
        "{\n\t.reg .pred pa;\n\t.reg .f32 ta;\n\t"
        "setp.ne.b32 pa, %3, 0;\n\t"
        "@pa ld.shared.f32 ta, [%0];\n\t@pa fma.rn.f32 ta, %1, %2, ta;\n\t@pa st.shared.f32 [%0], ta;\n\t}"
        :: "r"(qa), "f"(va), "f"(w), "r"(oka) : "memory");
}

// (-0 mode: the marker is -0.0, which the first fma replaces by the product itself)
template <bool NEG0>
__device__ __forceinline__ float upd(float old, float v, float w) {
    if (NEG0) return fmaf(v, w, old);
    return fmaf(v, w, __float_as_uint(old) == kAbsent ? 0.0f : old);
}

// The accumulate loop of one warp (output channel slice fixed by the round records): every
// work item (ic, input plane) of the staged chunk against the item's rounds {byte offset,
// weight}, read from shared memory by broadcast. Entries go 64 at a time, two per lane, so that
// two independent read-modify-writes are in flight per round. Entries of one item have distinct
// positions, so the 64 targets of a round are distinct; rounds are separated by __syncwarp (a
// later round may read what an earlier one wrote). Idle lanes address a safe interior word
// (every round offset keeps it inside the slice) and do not store.
// One work descriptor as a warp needs it: its round range and the lane's two entries.
struct FwdDesc {
    int r0, r1;          // rounds (records) of (oc, item)
    uint32_t aA, aB;     // accumulator byte addresses of the lane's entries (safe word when idle)
    float vA, vB;
    int n;               // entries of the descriptor (<= 64)
    int2 rr;             // REGREC: record r0 + lane (rounds broadcast by shuffles)
};

// REGREC (round records in global memory, large filter banks): lane j also fetches record
// r0 + j of the descriptor, so that its rounds read their records with shuffles instead of
// dependent L1 loads (the descriptor is prefetched one ahead, so the fetch latency is hidden)
template <bool REGREC>
__device__ __forceinline__ FwdDesc load_desc(uint32_t wdsc, int lane, uint32_t accs, uint32_t safe,
                                             const int* roffw, const uint32_t* spos, const float* sval,
                                             const int2* rec) {
    FwdDesc d;
    const int item = (int)(wdsc >> 19);
    d.r0 = roffw[item];
    d.r1 = roffw[item + 1];
    d.rr = make_int2(0, 0);
    if (REGREC && lane < d.r1 - d.r0) d.rr = rec[d.r0 + lane];
    const int s = (int)(wdsc & 0xfffu);
    d.n = (int)((wdsc >> 12) & 0x7fu);
    const bool okA = lane < d.n, okB = lane + 32 < d.n;
    d.aA = accs + (okA ? spos[s + lane] : safe);
    d.vA = okA ? sval[s + lane] : 0.0f;
    d.aB = accs + (okB ? spos[s + 32 + lane] : safe);
    d.vB = okB ? sval[s + 32 + lane] : 0.0f;
    return d;
}

// The accumulate loop of one warp (output channel slice fixed by the round records): every
// work item (ic, input plane) of the staged chunk against the item's rounds {byte offset,
// weight}, read from shared memory by broadcast. Entries go 64 at a time, two per lane, so that
// two independent read-modify-writes are in flight per round. Entries of one item have distinct
// positions, so the 64 targets of a round are distinct; rounds are separated by __syncwarp (a
// later round may read what an earlier one wrote). Idle lanes address a safe interior word
// (every round offset keeps it inside the slice) and do not store. The next descriptor's
// dependent shared loads (descriptor -> round range, entries) are issued before the current
// descriptor's rounds run.
template <bool NEG0, bool REGREC, bool PRED>
__device__ __forceinline__ void fwd_items(int nwork, int lane, uint32_t accs, uint32_t safe, const uint32_t* work,
                                          const int* roffw, const int2* rec, const uint32_t* spos,
                                          const float* sval, int2* wrec, uint32_t slo, uint32_t slen) {
    // a target outside the warp's band slice [slo, slo + slen) (an update from a halo input row
    // that leaves the band) is predicated off
    auto in_band = [&](uint32_t q) { return PRED ? (int)((q - slo) < slen) : 1; };
    if (nwork <= 0) return;
    FwdDesc nx = load_desc<REGREC>(work[0], lane, accs, safe, roffw, spos, sval, rec);
#pragma unroll 1
    for (int g = 0; g < nwork; ++g) {
        const FwdDesc d = nx;
        if (g + 1 < nwork) nx = load_desc<REGREC>(work[g + 1], lane, accs, safe, roffw, spos, sval, rec);
        if (d.r0 == d.r1) continue;
        const bool okA = lane < d.n, okB = lane + 32 < d.n;
        if (REGREC && d.r1 - d.r0 <= 32) {
            // the descriptor's records (fetched with its prefetch) go to the warp's shared buffer
            // now that they have arrived; the rounds read them by broadcast
            const int nr = d.r1 - d.r0;
            if (lane < nr) wrec[lane] = d.rr;
            __syncwarp();
            if (d.n > 32) {
#pragma unroll 2
                for (int r = 0; r < nr; ++r) {
                    const int2 q = wrec[r];
                    const uint32_t qa = d.aA + (uint32_t)q.x, qb = d.aB + (uint32_t)q.x;
                    const float w = __int_as_float(q.y);
                    if (NEG0) {
                        rmw2_neg0(qa, qb, d.vA, d.vB, w, okA & in_band(qa), okB & in_band(qb));
                    } else {
                        float oa = 0.0f, ob = 0.0f;
                        const bool pa = okA && in_band(qa), pb = okB && in_band(qb);
                        if (pa) oa = lds_u(qa);
                        if (pb) ob = lds_u(qb);
                        if (pa) sts_u(qa, upd<NEG0>(oa, d.vA, w));
                        if (pb) sts_u(qb, upd<NEG0>(ob, d.vB, w));
                    }
#ifndef SPC_NO_SYNCWARP
                    __syncwarp();
#endif
                }
            } else {
#pragma unroll 2
                for (int r = 0; r < nr; ++r) {
                    const int2 q = wrec[r];
                    const uint32_t qa = d.aA + (uint32_t)q.x;
                    const float w = __int_as_float(q.y);
                    if (NEG0) rmw1_neg0(qa, d.vA, w, okA & in_band(qa));
                    else if (okA && in_band(qa)) sts_u(qa, upd<NEG0>(lds_u(qa), d.vA, w));
#ifndef SPC_NO_SYNCWARP
                    __syncwarp();
#endif
                }
            }
            __syncwarp();   // (the buffer is rewritten by the next descriptor)
            continue;
        }
        if (d.n > 32) {
            int2 q = rec[d.r0];
#pragma unroll 2
            for (int r = d.r0; r < d.r1; ++r) {
                const int2 qn = rec[r + 1];   // next record in flight during this round (rec has a spare slot)
                const uint32_t qa = d.aA + (uint32_t)q.x, qb = d.aB + (uint32_t)q.x;
                const float w = __int_as_float(q.y);
                if (NEG0) {
                    rmw2_neg0(qa, qb, d.vA, d.vB, w, okA & in_band(qa), okB & in_band(qb));
                } else {
                    float oa = 0.0f, ob = 0.0f;   // idle lanes do not touch shared memory (racecheck-clean)
                    const bool pa = okA && in_band(qa), pb = okB && in_band(qb);
                    if (pa) oa = lds_u(qa);
                    if (pb) ob = lds_u(qb);
                    if (pa) sts_u(qa, upd<NEG0>(oa, d.vA, w));
                    if (pb) sts_u(qb, upd<NEG0>(ob, d.vB, w));
                }
#ifndef SPC_NO_SYNCWARP
                __syncwarp();
#endif
                q = qn;
            }
        } else {
            int2 q = rec[d.r0];
#pragma unroll 2
            for (int r = d.r0; r < d.r1; ++r) {
                const int2 qn = rec[r + 1];
                const uint32_t qa = d.aA + (uint32_t)q.x;
                if (NEG0) rmw1_neg0(qa, d.vA, __int_as_float(q.y), okA & in_band(qa));
                else if (okA && in_band(qa)) sts_u(qa, upd<NEG0>(lds_u(qa), d.vA, __int_as_float(q.y)));
#ifndef SPC_NO_SYNCWARP
                __syncwarp();
#endif
                q = qn;
            }
        }
    }
}

// One CTA = (b, output x-plane, band of TY rows, group of ocg output channels); its slice of the
// paper's temporary dense buffer lives in shared memory as [ocg][TY + 4hy rows][ZR
// columns] (2hy margin rows on each side catch the targets of halo inputs that fall outside the
// band). The stored inputs of every work item (ic, input plane x + dx - hx), rows of the band
// plus halo, are contiguous key runs (row index); they are staged once per CTA as (byte position,
// value) and shared by all warps. Warp w owns output channel oc0 + w: no two warps write the
// same word, no atomics, and a fixed order makes the result deterministic.
// EPI: kEpiSample -- the sampled pass (score histogram only); kEpiCand -- the main pass
// (candidate runs); kEpiRedo -- the main pass again, for the queued samples only, with every
// support entry of a failed segment as a candidate.
constexpr int kEpiSample = 1, kEpiCand = 2, kEpiRedo = 3;

template <bool REC_SMEM, bool PRED, int EPI>
__device__ __forceinline__ void fwd_tile(const Geo& gx, const Geo& gy, const KGeo& kg, const FwdTile& t,
                                         const FwdArgs& a, int64_t bl, int tin) {
    extern __shared__ __align__(16) float smf[];
    const int c_in = (int)gx.C, c_out = (int)gy.C;
    const int Z = gy.Z, ZR = t.ZR;
    const int P = (int)fdiv((uint32_t)tin, t.fd_nty);   // output plane (w, x): P = w*X + x
    const int ty = tin - P * t.nty;
    const int wpl = (int)fdiv((uint32_t)P, t.fd_X), x = P - wpl * gy.X;
    const int64_t b = a.b0 + bl;                        // global sample (input rows)
    const int oc0 = blockIdx.y * t.ocg;
    const int nocl = min(t.ocg, c_out - oc0);
    const int y0 = ty * t.TY, ye = min(y0 + t.TY, gy.Y);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int SL = t.RA * ZR;                        // floats per output-channel slice
    const int PK = t.PK;

    // shared layout: acc [ocg*SL] | spos [cap] | sval [cap] | ioff | iglob | ibase | work | misc |
    // rpair [ocg*PK] | rec [nwg]
    float* acc = smf;
    uint32_t* spos = reinterpret_cast<uint32_t*>(smf + (size_t)t.ocg * SL);
    float* sval = reinterpret_cast<float*>(spos + kStageCap);
    int* ioff = reinterpret_cast<int*>(sval + kStageCap);
    uint32_t* iglob = reinterpret_cast<uint32_t*>(ioff + r4(PK + 1));
    uint32_t* ibase = iglob + r4(PK + 1);
    int* wpre = reinterpret_cast<int*>(ibase + r4(PK + 1));   // first work descriptor of each item
    uint32_t* work = reinterpret_cast<uint32_t*>(wpre + r4(PK + 1));
    uint32_t* misc = work + r4(kStageCap / 64 + PK + 1);
    int2* rpair = reinterpret_cast<int2*>(misc + 80);   // misc: 80 words (u64 block-scan scratch)
    int2* rec = rpair + (size_t)t.ocg * PK;
    const int2* recp = REC_SMEM ? rec : a.rnd + (int64_t)blockIdx.y * t.nwg_max;
    uint32_t* hist = spos;                           // epilogue only

    const bool neg0 = *a.guard == 0;                 // -0 accumulation mode (value_guard_kernel)
    const uint32_t marker = neg0 ? kNegZero : kAbsent;
    // ---- prologue. The global loads go out first (round offsets / records by cp.async, item
    // bounds into registers) so that their latency overlaps the accumulator fill.
    int* roffs = reinterpret_cast<int*>(rpair);      // raw round offsets of the group [ocg*PK + 1]
    {
        const int* groff = a.roff + (int64_t)blockIdx.y * (t.ocg * PK + 1);
        const uint32_t rs = (uint32_t)__cvta_generic_to_shared(roffs);
        for (int i = threadIdx.x; i <= t.ocg * PK; i += blockDim.x)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(rs + 4u * i), "l"(groff + i) : "memory");
        if (REC_SMEM) {
            const int2* grec = a.rnd + (int64_t)blockIdx.y * t.nwg_max;
            const uint32_t rcs = (uint32_t)__cvta_generic_to_shared(rec);
            for (int i = threadIdx.x; i < t.nwg_max; i += blockDim.x)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(rcs + 8u * i), "l"(grec + i) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // work items: stored inputs of (ic, plane xs), rows ylo..yhi-1 -> one contiguous key run
    const int ylo = max(0, y0 - kg.hy), yhi = min(gy.Y, ye + kg.hy);
    auto item_bounds = [&](int q, uint32_t& e0, uint32_t& n, uint32_t& rb) {
        e0 = n = rb = 0u;
        if (q >= PK) return;
        const int KWX = kg.kw * kg.kx;
        const int ic = q / KWX, it = q - ic * KWX;
        const int ws = wpl + it / kg.kx - kg.hw, xs = x + it % kg.kx - kg.hx;   // input plane (w, x)
        if (ws >= 0 && ws < gx.W && xs >= 0 && xs < gx.X) {
            const int64_t row = (((b * c_in + ic) * gx.W + ws) * gx.X + xs) * (int64_t)gx.Y + ylo;
            e0 = a.xrow[row];
            n = a.xrow[row + (yhi - ylo)] - e0;
            rb = (uint32_t)((uint64_t)row * (uint64_t)Z);   // low word of the row's first key
        }
    };
    uint32_t pe0 = 0, pn = 0, prb = 0;
    item_bounds(threadIdx.x, pe0, pn, prb);          // first batch of items, loads in flight
    {
        const int n4 = t.ocg * SL / 4;
        const uint4 ab = make_uint4(marker, marker, marker, marker);
        for (int i = threadIdx.x; i < n4; i += blockDim.x) reinterpret_cast<uint4*>(smf)[i] = ab;
    }
    // item entry offsets and work-descriptor offsets (groups of <= 64 entries) by one scan of
    // (count << 32 | groups)
    uint64_t carry = 0;
    for (int q0 = 0; q0 < PK; q0 += blockDim.x) {
        const int q = q0 + threadIdx.x;
        uint32_t e0 = pe0, n = pn, rb = prb;
        if (q0 > 0) item_bounds(q, e0, n, rb);
        const uint64_t packed = ((uint64_t)n << 32) | (uint64_t)((n + 63) >> 6);
        uint64_t tot;
        const uint64_t ex = block_excl_scan(packed, reinterpret_cast<uint64_t*>(misc), &tot);
        if (q < PK) {
            ioff[q] = (int)((carry + ex) >> 32);
            wpre[q] = (int)((carry + ex) & 0xffffffffu);
            iglob[q] = e0;
            ibase[q] = rb;
        }
        carry += tot;
    }
    if (threadIdx.x == 0) ioff[PK] = (int)(carry >> 32);
    const int total = (int)(carry >> 32);
    const int wtotal = (int)(carry & 0xffffffffu);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();

    const uint32_t accs = (uint32_t)__cvta_generic_to_shared(acc);
    const int mrow = PRED ? 0 : 2 * kg.hy;           // margin rows below the band
    const uint32_t safe = (uint32_t)(mrow * ZR + t.cz) * 4u;   // a word of slice 0 (idle lanes never access it)
    const float invZ = 1.0f / (float)Z;
    // accumulator row of input row ylo (input row yi -> row yi - (y0 - 2hy))
    const int arow0 = ylo - y0 + mrow;   // (pred mode: -hy for a halo below, rows below the slice)
    const bool single = total <= kStageCap;          // the usual case: one chunk, descriptors known
    for (int f0 = 0; f0 < total; f0 += kStageCap) {
        const int f1 = min(total, f0 + kStageCap);
        // ---- stage the chunk: (byte position in a channel slice, value). The items' key runs
        // are one concatenated list; thread i takes list positions i, i + 256, ... (item by a
        // binary search over the item offsets), all key / value loads of a batch of eight in
        // flight before any is used.
        {
            constexpr int kJ = 8;
            for (int base = f0 + (int)threadIdx.x; base < f1; base += kFwdThreads * kJ) {
                uint32_t kw[kJ], rbj[kJ];
                float vj[kJ];
                int dj[kJ];
#pragma unroll
                for (int j = 0; j < kJ; ++j) {
                    const int pos = base + kFwdThreads * j;
                    dj[j] = -1;
                    kw[j] = 0u;
                    rbj[j] = 0u;
                    vj[j] = 0.0f;
                    if (pos < f1) {
                        int lo = 0, hi = PK;   // last item q with ioff[q] <= pos
                        while (hi - lo > 1) {
                            const int mid = (lo + hi) >> 1;
                            if (ioff[mid] <= pos) lo = mid; else hi = mid;
                        }
                        const uint32_t e = iglob[lo] + (uint32_t)(pos - ioff[lo]);
                        kw[j] = a.xkeys.lo(e);   // low word of the key
                        vj[j] = a.xvals[e];
                        rbj[j] = ibase[lo];
                        dj[j] = pos - f0;
                    }
                }
#pragma unroll
                for (int j = 0; j < kJ; ++j) {
                    if (dj[j] < 0) continue;
                    const uint32_t L = kw[j] - rbj[j];   // < 2^32: offset within the run
                    const uint32_t yrel = div_small(L, (uint32_t)Z, invZ);
                    const uint32_t z = L - yrel * (uint32_t)Z;
                    spos[dj[j]] = (uint32_t)(((int)yrel + arow0) * ZR + (int)z + t.cz) * 4u;   // (mod 2^32)
                    sval[dj[j]] = vj[j];
                }
            }
        }
        if (single)   // work descriptors of item q by thread q
            for (int pk = threadIdx.x; pk < PK; pk += kFwdThreads) {
                const int s0 = ioff[pk], s1 = ioff[pk + 1];
                for (int gi = 0; 64 * gi < s1 - s0; ++gi) {
                    const int st = s0 + 64 * gi;
                    work[wpre[pk] + gi] = (uint32_t)st | ((uint32_t)min(64, s1 - st) << 12) | ((uint32_t)pk << 19);
                }
            }
        __syncthreads();
        if (!single) {
            if (warp == 0) {   // work list of the chunk: groups of <= 64 entries of one item
                int wcar = 0;
                for (int p0 = 0; p0 < PK; p0 += 32) {
                    const int pk = p0 + lane;
                    int s0 = 0, s1 = 0;
                    if (pk < PK) {
                        s0 = max(ioff[pk], f0) - f0;
                        s1 = min(ioff[pk + 1], f1) - f0;
                    }
                    const int ng = s1 > s0 ? (s1 - s0 + 63) >> 6 : 0;
                    const int inc = warp_incl_scan(ng);
                    for (int gi = 0; gi < ng; ++gi) {
                        const int st = s0 + 64 * gi;
                        work[wcar + inc - ng + gi] = (uint32_t)st | ((uint32_t)min(64, s1 - st) << 12) | ((uint32_t)pk << 19);
                    }
                    wcar += __shfl_sync(kFull, inc, 31);
                }
                if (lane == 0) misc[0] = (uint32_t)wcar;
            }
            __syncthreads();
        }
        const int nwork = single ? wtotal : (int)misc[0];
        const uint32_t slo = accs + (uint32_t)(warp * SL) * 4u, slen = (uint32_t)SL * 4u;   // this warp's slice
        // ---- accumulate (Alg. 1 inner loops)
        if (warp < nocl) {
            if (neg0)
                fwd_items<true, !REC_SMEM, PRED>(nwork, lane, accs, safe, work, roffs + warp * PK, recp, spos, sval,
                                           rec + warp * 32, slo, slen);
            else
                fwd_items<false, !REC_SMEM, PRED>(nwork, lane, accs, safe, work, roffs + warp * PK, recp, spos, sval,
                                            rec + warp * 32, slo, slen);
        }
        __syncthreads();
    }

    // ------------------------------------------------------------------------ epilogue
    const int nyr = ye - y0;
    if (EPI != kEpiSample) {
        // "get non-zero entries" / "add bias" / candidates for "select k largest"
        // (P:80): warp w reads only its own channel's slice, so no barrier is needed
        if (warp >= nocl) return;
        const int oc = oc0 + warp;
        const int64_t s = bl * c_out + oc;
        if (EPI == kEpiRedo && !a.fail[s]) return;
        const float bv = a.bias ? __ldg(&a.bias[oc]) : 0.0f;
        const float* S = acc + warp * SL + mrow * ZR + t.cz;
        const uint32_t tl = EPI == kEpiRedo ? 0u : a.tlow[s];
        const uint32_t pbase = (uint32_t)(((int64_t)P * gy.Y + y0) * Z);
        uint32_t* cp = a.cpos + s * gy.V + pbase;
        float* cv = a.cval + s * gy.V + pbase;
        uint32_t n, mx;
        static_assert(kFwdWarps * kCandBuf <= kStageCap, "candidate buffers live in the staging area");
        uint2* bp = reinterpret_cast<uint2*>(spos) + warp * kCandBuf;   // (spos | sval: 8 B per staged entry)
        const bool full = (Z & 127) == 0;
        if (a.attn == SPC_ATTN_MAGNITUDE) {
            if (full) epi_cand<SPC_ATTN_MAGNITUDE, true>(S, nyr, Z, ZR, bv, tl, marker, pbase, cp, cv, bp, n, mx);
            else epi_cand<SPC_ATTN_MAGNITUDE, false>(S, nyr, Z, ZR, bv, tl, marker, pbase, cp, cv, bp, n, mx);
        } else if (a.attn == SPC_ATTN_RAW) {
            if (full) epi_cand<SPC_ATTN_RAW, true>(S, nyr, Z, ZR, bv, tl, marker, pbase, cp, cv, bp, n, mx);
            else epi_cand<SPC_ATTN_RAW, false>(S, nyr, Z, ZR, bv, tl, marker, pbase, cp, cv, bp, n, mx);
        } else {
            epi_cand<SPC_ATTN_NONE, false>(S, nyr, Z, ZR, bv, tl, marker, pbase, cp, cv, bp, n, mx);
        }
        if (lane == 0) {
            a.tcnt[s * a.ntile + tin] = n;
            if (n) {
                atomicAdd(&a.cand_cur[s], (unsigned long long)n);
                atomicMax(&a.cmax[s], mx);
            }
        }
        return;
    }
    // sampled pass: the tile's score histogram per output channel, merged into the segment's
    // (support size = its total). Two histogram buffers alternate between output channels -- A in
    // the staging area, B in the accumulator slice of the first channel once that is consumed --
    // so a channel's histogram is flushed while the next channel's rows are being binned.
    constexpr int kHist4 = (kSelBins + 32) / 4;      // bins + one dummy bin per lane
    const bool dbuf = nocl > 1 && SL >= 4 * kHist4;
    uint4* histA = reinterpret_cast<uint4*>(hist);
    uint4* histB = reinterpret_cast<uint4*>(acc);
    for (int i = threadIdx.x; i < kHist4; i += blockDim.x) histA[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    for (int ocl = 0; ocl < nocl; ++ocl) {
        const int oc = oc0 + ocl;
        const int64_t s = bl * c_out + oc;
        const float bv = a.bias ? __ldg(&a.bias[oc]) : 0.0f;
        const float* S = acc + ocl * SL + mrow * ZR + t.cz;
        uint4* hist4 = (dbuf && (ocl & 1)) ? histB : histA;
        const uint32_t hist_s = (uint32_t)__cvta_generic_to_shared(hist4);
        if (a.attn == SPC_ATTN_RAW) epi_hist_rows<SPC_ATTN_RAW>(S, bv, nyr, Z, ZR, hist_s, marker);
        else epi_hist_rows<SPC_ATTN_MAGNITUDE>(S, bv, nyr, Z, ZR, hist_s, marker);
        __syncthreads();
        if (dbuf && ocl == 0) {   // slice 0 is consumed: it becomes buffer B
            for (int i = threadIdx.x; i < kHist4; i += blockDim.x) histB[i] = make_uint4(0u, 0u, 0u, 0u);
            __syncthreads();
        }
        uint32_t* gh = a.hist + s * kSelBins;
        for (int i = threadIdx.x; i < kHist4; i += blockDim.x) {
            const uint4 h = hist4[i];
            if (h.x | h.y | h.z | h.w) {
                hist4[i] = make_uint4(0u, 0u, 0u, 0u);
                if (4 * i < kSelBins) {
                    // two adjacent bins per 64-bit atomic (a bin's total is at most V < 2^32, so
                    // the low word never carries into the high one)
                    unsigned long long* g2 = reinterpret_cast<unsigned long long*>(gh + 4 * i);
                    if (h.x | h.y) atomicAdd(g2, (unsigned long long)h.x | ((unsigned long long)h.y << 32));
                    if (h.z | h.w) atomicAdd(g2 + 1, (unsigned long long)h.z | ((unsigned long long)h.w << 32));
                }
            }
        }
        if (!dbuf) __syncthreads();   // single buffer: the next channel bins only after the flush
    }
}

// One CTA = one tile (b, x, band, output-channel group): main pass (EPI = kEpiCand), grid
// (B * ntile, n_ocg).
template <bool REC_SMEM, bool PRED>
__global__ void __launch_bounds__(kFwdThreads, 2) conv_fwd_kernel(Geo gx, Geo gy, KGeo kg, FwdTile t, FwdArgs a) {
    const uint32_t tile = blockIdx.x, bl = fdiv(tile, a.fd_ntile);   // (B * ntile < 2^31)
    fwd_tile<REC_SMEM, PRED, kEpiCand>(gx, gy, kg, t, a, bl, (int)(tile - bl * (uint32_t)a.ntile));
}

// Sampled pass: grid (B * nsamp, n_ocg); tile j of a segment's sample = j*sp_period + sp_off.
template <bool REC_SMEM, bool PRED>
__global__ void __launch_bounds__(kFwdThreads, 2) conv_fwd_sample_kernel(Geo gx, Geo gy, KGeo kg, FwdTile t,
                                                                         FwdArgs a) {
    const uint32_t j = blockIdx.x, bl = fdiv(j, a.fd_nsamp);
    fwd_tile<REC_SMEM, PRED, kEpiSample>(gx, gy, kg, t, a, bl, (int)(j - bl * (uint32_t)a.nsamp) * a.sp_period + a.sp_off);
}

// Redo pass: grid (ntile, n_ocg); block t recomputes tile t of every queued sample (normally
// none: the block exits at once).
template <bool REC_SMEM, bool PRED>
__global__ void __launch_bounds__(kFwdThreads, 2) conv_fwd_redo_kernel(Geo gx, Geo gy, KGeo kg, FwdTile t,
                                                                       FwdArgs a) {
    const int nq = *a.redo_n;
    for (int i = 0; i < nq; ++i) {
        fwd_tile<REC_SMEM, PRED, kEpiRedo>(gx, gy, kg, t, a, a.redo_b[i], (int)blockIdx.x);
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

// exclusive scan of a per-segment u64 array (single block); total -> *total. add_base: the scan
// starts at the value *total holds on entry (appending passes), and *total grows by the sum.
__global__ void seg_scan_u64_kernel(const uint64_t* in, uint64_t* out, int64_t n, int64_t* total, int add_base = 0) {
    __shared__ uint64_t sm[33];
    uint64_t carry = add_base ? (uint64_t)*total : 0;   // read by all before the first barrier
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

// two independent segment scans in one launch (candidate and staging offsets)
__global__ void seg_scan2_u64_kernel(const uint64_t* in, uint64_t* out, const uint64_t* in2, uint64_t* out2, int64_t n) {
    __shared__ uint64_t sm[33];
    for (int pass = 0; pass < 2; ++pass) {
        const uint64_t* src = pass ? in2 : in;
        uint64_t* dst = pass ? out2 : out;
        if (!src) continue;   // block-uniform
        uint64_t carry = 0;
        for (int64_t base = 0; base < n; base += blockDim.x) {
            const int64_t i = base + threadIdx.x;
            const uint64_t v = i < n ? src[i] : 0;
            uint64_t t;
            const uint64_t ex = block_excl_scan(v, sm, &t);
            if (i < n) dst[i] = carry + ex;
            carry += t;
        }
        if (threadIdx.x == 0) dst[n] = carry;
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
    {
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

// f(e) for every candidate e of a segment's list, four independent loads in flight per thread
template <typename F>
__device__ __forceinline__ void for_cands(const uint2* __restrict__ c, uint64_t n, F f) {
    uint64_t i = threadIdx.x;
    for (; i + 3 * kResThreads < n; i += 4 * kResThreads) {
        const uint2 e0 = c[i], e1 = c[i + kResThreads], e2 = c[i + 2 * kResThreads], e3 = c[i + 3 * kResThreads];
        f(e0);
        f(e1);
        f(e2);
        f(e3);
    }
    for (; i < n; i += kResThreads) f(c[i]);
}
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
    if (n <= (uint64_t)kResThreads) {
        // small candidate sets (e.g. the 784-voxel MNIST-like segments): the `need`-th largest
        // composite key directly by ranking -- each key counts the keys above it (all distinct)
        for (uint32_t i = threadIdx.x; i < (uint32_t)n; i += blockDim.x) {
            const uint2 e = c[i];
            sc[i] = composite(score_bits(e.y, a.attn), e.x);
        }
        __syncthreads();
        const uint64_t want = (uint64_t)st.need - 1;   // rank (0 = largest) of kstar
        for (uint32_t i = threadIdx.x; i < (uint32_t)n; i += blockDim.x) {
            const uint64_t k = sc[i];
            uint32_t above = 0;
            for (uint32_t j = 0; j < (uint32_t)n; ++j) above += sc[j] > k ? 1u : 0u;
            if (above == want) sh_prefix = k;
        }
        __syncthreads();
        const uint64_t kstar = sh_prefix;
        if (threadIdx.x == 0) {
            st.kstar = kstar;
            a.seg[s] = st;
        }
        for (uint32_t i = threadIdx.x; i < (uint32_t)n; i += blockDim.x) {   // aggregated per chunk in the warp
            const bool sel = sc[i] >= kstar;
            const uint32_t ch = sel ? (uint32_t)(~sc[i]) / kChunk : 0xffffffffu;
            const unsigned grp = __match_any_sync(__activemask(), ch);
            if (sel && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&a.tile_sel[s * a.nchunk + ch], (uint32_t)__popc(grp));
        }
        return;
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
            for_cands(c, n, [&](uint2 e) {
                const uint64_t k = composite(score_bits(e.y, a.attn), e.x);
                if ((k & mask) == prefix) atomicAdd(&h[(uint32_t)(k >> sh) & dmask], 1u);
            });
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
            for_cands(c, n, [&](uint2 e) {
                const uint64_t k = composite(score_bits(e.y, a.attn), e.x);
                if ((k & m2) == p2) sc[atomicAdd(&sh_ns, 1u)] = k;
            });
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
    // selected candidates per chunk; a chunk's candidates sit together in the list (classify
    // appends them as one run), so the lanes of a warp aggregate their counts per chunk first
    const int lane = threadIdx.x & 31;
    uint32_t* tsel = a.tile_sel + s * a.nchunk;
    for_cands(c, n, [&](uint2 e) {
        const bool sel = composite(score_bits(e.y, a.attn), e.x) >= kstar;
        const uint32_t ch = sel ? e.x / kChunk : 0xffffffffu;
        const unsigned grp = __match_any_sync(__activemask(), ch);
        if (sel && lane == __ffs(grp) - 1) atomicAdd(&tsel[ch], (uint32_t)__popc(grp));
    });
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
    const uint64_t kb = ((uint64_t)a.seg0 + (uint64_t)s) * (uint64_t)V;
    // composite(score, p) = (score << 32 | ~p) >= kstar, as two 32-bit compares
    const uint32_t ks = (uint32_t)(st.kstar >> 32), kp = (uint32_t)st.kstar;
    for (uint32_t i0 = 0; i0 < n; i0 += 128) {   // four groups of 32 loaded before any is used
        uint2 e[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const uint32_t i = i0 + 32u * g + lane;
            e[g] = i < n ? in[i] : make_uint2(0u, kAbsent);
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const bool ok = i0 + 32u * g + lane < n;
            const uint32_t sc = score_bits(e[g].y, a.attn);
            const bool keep = ok && (st.keep_all || sc > ks || (sc == ks && ~e[g].x >= kp));
            const unsigned m = __ballot_sync(kFull, keep);
            if (keep) {
                const uint64_t q = out + __popc(m & ((1u << lane) - 1u));
                a.out_keys.put(q, kb + e[g].x);
                a.out_vals[q] = __uint_as_float(e[g].y);
            }
            out += __popc(m);
        }
    }
}

cudaError_t launch_seg_scan_u64(const uint64_t* in, uint64_t* out, int64_t n, int64_t* total, int add_base,
                                cudaStream_t s) {
    SPC_PHASE("seg_scan", s, 1);
    seg_scan_u64_kernel<<<1, 1024, 0, s>>>(in, out, n, total, add_base);
    return cudaGetLastError();
}

void plan_fwd_sampling(const Geo& gy, const FwdTile& t, int attn, FwdArgs* a) {
    a->ntile = (int)((int64_t)gy.W * gy.X * t.nty);
    // every sp_period-th tile of a segment: for large segments the largest prime in 37..61 that
    // leaves at least 16 sampled tiles, else the largest prime <= 31 that leaves at least 8 --
    // never one dividing the band count (the sampled tiles cycle through the bands); no sampling
    // for small segments or without attention
    static const int big[] = {61, 59, 53, 47, 43, 41, 37};
    static const int small[] = {31, 29, 23, 19, 17, 13, 11, 7, 5, 3};
    int P = 0;
    for (int p : big)
        if (a->ntile >= 16 * p && t.nty % p != 0) { P = p; break; }
    if (P == 0)
        for (int p : small)
            if (a->ntile >= 8 * p && t.nty % p != 0) { P = p; break; }
    a->sp_period = P > 0 ? P : 1;
    a->sp_off = P / 2;
    a->nsamp = (attn != SPC_ATTN_NONE && P > 0) ? (a->ntile - a->sp_off + P - 1) / P : 0;
    a->fd_ntile = make_fastdiv((uint32_t)a->ntile);
    a->fd_nsamp = make_fastdiv((uint32_t)std::max(1, a->nsamp));
}

template <bool REC, bool PRED>
static cudaError_t set_fwd_smem(size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(conv_fwd_kernel<REC, PRED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(conv_fwd_sample_kernel<REC, PRED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(conv_fwd_redo_kernel<REC, PRED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return e;
}

template <bool REC, bool PRED>
static void launch_fwd_passes(const Geo& gx, const Geo& gy, const KGeo& kg, const FwdTile& t, const FwdArgs& a,
                              int which, cudaStream_t s) {
    if (which == 0) {
        const dim3 grid((unsigned)(gy.B * a.nsamp), (unsigned)t.n_ocg);
        SPC_PHASE("conv_fwd_sample", s, 1);
        conv_fwd_sample_kernel<REC, PRED><<<grid, kFwdThreads, t.smem, s>>>(gx, gy, kg, t, a);
    } else if (which == 1) {
        const dim3 grid((unsigned)(gy.B * a.ntile), (unsigned)t.n_ocg);
        SPC_PHASE("conv_fwd", s, 1);
        conv_fwd_kernel<REC, PRED><<<grid, kFwdThreads, t.smem, s>>>(gx, gy, kg, t, a);
    } else {
        const dim3 grid((unsigned)a.ntile, (unsigned)t.n_ocg);
        SPC_PHASE("conv_fwd_redo", s, 1);
        conv_fwd_redo_kernel<REC, PRED><<<grid, kFwdThreads, t.smem, s>>>(gx, gy, kg, t, a);
    }
}

cudaError_t launch_conv_fwd_stream(const Geo& gx, const Geo& gy, const KGeo& kg, const FwdTile& t,
                                   const FwdArgs& a, cudaStream_t s) {
    const int64_t nseg = gy.B * gy.C;
    if (nseg == 0) return a.out_append ? cudaSuccess : cudaMemsetAsync(a.out_nnz, 0, sizeof(int64_t), s);
    cudaError_t e = t.rec_smem ? (t.pred ? set_fwd_smem<true, true>(t.smem) : set_fwd_smem<true, false>(t.smem))
                               : (t.pred ? set_fwd_smem<false, true>(t.smem) : set_fwd_smem<false, false>(t.smem));
    if (e != cudaSuccess) return e;
    const size_t segb = sizeof(uint64_t) * (size_t)nseg;
    cudaMemsetAsync(a.seg_count, 0, segb, s);
    cudaMemsetAsync(a.cand_cur, 0, segb, s);
    cudaMemsetAsync(a.cmax, 0, sizeof(uint32_t) * (size_t)nseg, s);
    cudaMemsetAsync(a.fail, 0, sizeof(int) * (size_t)nseg, s);
    cudaMemsetAsync(a.bflag, 0, sizeof(int) * (size_t)gy.B, s);
    cudaMemsetAsync(a.redo_n, 0, sizeof(int), s);
    cudaMemsetAsync(a.tile_sel, 0, sizeof(uint32_t) * (size_t)(nseg * a.ntile), s);
    if (!a.out_append) {   // later passes of sparse_conv_fwd_pass reuse the guard and the rounds
        if (!a.guard_done) {
            cudaMemsetAsync(a.guard, 0, sizeof(int), s);
            SPC_PHASE("value_guard", s, 1);
            value_guard_kernel<<<num_sms() * 4, 256, 0, s>>>(a.xvals, a.x_nnz_dev, a.x_nnz, a.guard);
        }
        SPC_PHASE("fwd_rounds", s, 1);
        fwd_rounds_kernel<<<(unsigned)t.n_ocg, 256, 0, s>>>(kg, (int)gx.C, (int)gy.C, t, a.meta2, a.val2, a.off2,
                                                          a.rnd, a.roff, a.guard);
    }
    auto passes = [&](int which) {
        if (t.rec_smem) {
            if (t.pred) launch_fwd_passes<true, true>(gx, gy, kg, t, a, which, s);
            else launch_fwd_passes<true, false>(gx, gy, kg, t, a, which, s);
        } else {
            if (t.pred) launch_fwd_passes<false, true>(gx, gy, kg, t, a, which, s);
            else launch_fwd_passes<false, false>(gx, gy, kg, t, a, which, s);
        }
    };
    if (a.nsamp > 0) {
        cudaMemsetAsync(a.hist, 0, sizeof(uint32_t) * kSelBins * (size_t)nseg, s);
        passes(0);
        e = launch_stream_find(a, s);
        if (e != cudaSuccess) return e;
    } else {
        cudaMemsetAsync(a.tlow, 0, sizeof(uint32_t) * (size_t)nseg, s);
    }
    // test hook: a threshold above every score, so that every non-empty segment takes the redo
    // path (tests/test_parity_gpu.py::test_fwd_forced_redo)
    if (const char* f = getenv("SPC_FWD_FORCE_REDO"))
        if (f[0] == '1') cudaMemsetAsync(a.tlow, 0xff, sizeof(uint32_t) * (size_t)nseg, s);
    passes(1);
    e = launch_stream_resolve(gy, t, a, 0, s);
    if (e != cudaSuccess) return e;
    passes(2);
    e = launch_stream_resolve(gy, t, a, 1, s);
    if (e != cudaSuccess) return e;
    e = launch_stream_tail(gy, t, a, s);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_conv_fwd_pipeline(const Geo& gx, const Geo& gy, const KGeo& kg, const FwdTile& t,
                                     const FwdArgs& a, cudaStream_t s, const GemmPlan* gp, const GemmArgs* ga) {
    const int64_t nseg = gy.B * gy.C;
    if (nseg == 0) return a.out_append ? cudaSuccess : cudaMemsetAsync(a.out_nnz, 0, sizeof(int64_t), s);
    if (!gp || !ga) return cudaErrorInvalidValue;   // variant S runs launch_conv_fwd_stream
    const size_t segb = sizeof(uint64_t) * (size_t)nseg;
    cudaMemsetAsync(a.seg_count, 0, segb, s);
    cudaMemsetAsync(a.cand_cur, 0, segb, s);
    cudaMemsetAsync(a.stg_cur, 0, segb, s);
    cudaMemsetAsync(a.tile_sel, 0, sizeof(uint32_t) * (size_t)(nseg * a.nchunk), s);
    if (a.attn != SPC_ATTN_NONE) cudaMemsetAsync(a.hist, 0, sizeof(uint32_t) * kSelBins * (size_t)nseg, s);
    const unsigned sgrid = (unsigned)(nseg * a.nchunk);
    {
        cudaError_t eg = launch_conv_gemm(gx, gy, kg, *gp, *ga, a, s);
        if (eg != cudaSuccess) return eg;
    }
    { SPC_PHASE("fwd_find", s, 1); fwd_find_kernel<<<(unsigned)nseg, 256, 0, s>>>(a, nseg); }
    {
        SPC_PHASE("seg_scan", s, 1);
        seg_scan2_u64_kernel<<<1, 1024, 0, s>>>(a.attn != SPC_ATTN_NONE ? a.cand_cnt : nullptr, a.cand_off, a.stg_cnt,
                                               a.stg_off, nseg);
    }
    { SPC_PHASE("fwd_classify", s, 1); fwd_classify_kernel<<<sgrid, kChunkThreads, 0, s>>>(a, gy.V); }
    if (a.attn != SPC_ATTN_NONE) {
        SPC_PHASE("fwd_resolve", s, 1);
        fwd_resolve_kernel<<<(unsigned)nseg, kResThreads, 0, s>>>(a);
    }
    // kept per segment goes to cand_cnt (reused as scratch), then segment offsets
    { SPC_PHASE("fwd_chunk_scan", s, 1); fwd_chunk_scan_kernel<<<(unsigned)nseg, 256, 0, s>>>(a, a.cand_cnt); }
    { SPC_PHASE("seg_scan", s, 1); seg_scan_u64_kernel<<<1, 1024, 0, s>>>(a.cand_cnt, a.seg_off, nseg, a.out_nnz, a.out_append); }
    { SPC_PHASE("fwd_write", s, 1); fwd_write_kernel<<<(unsigned)((nseg * a.nchunk + kWriteWarps - 1) / kWriteWarps), 32 * kWriteWarps, 0, s>>>(a, gy.V); }
    return cudaGetLastError();
}

}  // namespace spc

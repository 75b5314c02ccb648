// Attention as a standalone layer: per (b, c) segment of a COO map keep the k
// entries with the largest score (|y| for variant (ii), y for variant (i)); ties go to the
// smaller key (reading R7). The fused forward has its own pipeline (conv_fwd.cu); this one
// serves attention_topk.
//
// One CTA per segment. Exact radix select on the order-preserving u32 score: up to three digit
// passes (11, 11, 10 bits) find the threshold T and the number `need` of entries with score == T
// that are kept. The first digit is counted over the segment's values; when its threshold bucket
// holds at most 8192 entries their scores are gathered into shared memory and the other digits
// run there (else over the values again, mostly L2 hits). A final pass compacts in key order -- score > T, or == T while fewer than `need` earlier ties were
// kept -- with coalesced loads and stores (one ballot per 32 entries, warp totals scanned across
// the block). Output offsets per segment are known before the select: min(n_s, k).
#include "spc_internal.cuh"
#include "block_scan.cuh"

namespace spc {

#ifndef SPC_TK_THREADS
#define SPC_TK_THREADS 256
#endif
constexpr int kTkThreads = SPC_TK_THREADS;
constexpr int kTkWarps = kTkThreads / 32;
constexpr int kTkG = 8;                                 // groups of 32 entries per warp and tile
constexpr uint32_t kTkTile = (uint32_t)kTkThreads * kTkG;
constexpr uint32_t kTkCand = 8192;                      // bucket scores kept in shared memory (32 KB)

// seg_off[s] = sum over earlier segments of kept(s') with kept = n_s if n_s <= k else k
__global__ void topk_offsets_kernel(const uint32_t* __restrict__ row_ptr, int64_t R, int64_t nseg, int64_t k,
                                    uint64_t* __restrict__ seg_off, int64_t* __restrict__ total) {
    __shared__ uint64_t sm[33];
    uint64_t carry = 0;
    for (int64_t base = 0; base < nseg; base += blockDim.x) {
        const int64_t s = base + threadIdx.x;
        uint64_t v = 0;
        if (s < nseg) {
            const uint64_t n = (uint64_t)(row_ptr[(s + 1) * R] - row_ptr[s * R]);
            v = n <= (uint64_t)k ? n : (uint64_t)k;
        }
        uint64_t t;
        const uint64_t ex = block_excl_scan(v, sm, &t);
        if (s < nseg) seg_off[s] = carry + ex;
        carry += t;
    }
    if (threadIdx.x == 0) *total = (int64_t)carry;
}

__global__ void __launch_bounds__(kTkThreads, 1024 / kTkThreads)
topk_seg_kernel(Keys keys, const float* __restrict__ vals, const uint32_t* __restrict__ row_ptr,
                int64_t R, int attn, int64_t k, const uint64_t* __restrict__ seg_off, KeysOut ok,
                float* __restrict__ ov, int64_t* __restrict__ osrc) {
    __shared__ uint32_t h[kSelBins];
    __shared__ uint32_t sm[33];
    __shared__ uint32_t wt[kTkWarps + 1], wk[kTkWarps + 1];
    __shared__ uint32_t sh_bin, sh_need, sh_cnt;
    __shared__ uint32_t cand[kTkCand];   // scores of the threshold bucket after the first digit
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t s = blockIdx.x;
    const uint32_t lo = row_ptr[s * R], hi = row_ptr[(s + 1) * R];
    const bool keep_all = (uint64_t)(hi - lo) <= (uint64_t)k;
    uint32_t T = 0, pmask = 0, need = 0;
    // one radix-select step over a histogram h of nb bins: the bin holding the need-th largest
    auto find_bin = [&](uint32_t nb) {
        const int per = (int)nb / kTkThreads;   // bins nb-1-per*t .. nb-per*(t+1) for thread t
        uint32_t own = 0;
        for (int q = 0; q < per; ++q) own += h[nb - 1 - per * tid - q];
        uint32_t tot;
        const uint32_t before = block_excl_scan(own, sm, &tot);
        if (before < need && before + own >= need) {
            uint32_t cum = before;
            for (int q = 0; q < per; ++q) {
                const uint32_t bin = nb - 1 - per * tid - q, hb = h[bin];
                if (cum + hb >= need) {
                    sh_bin = bin;
                    sh_need = need - cum;
                    sh_cnt = hb;
                    break;
                }
                cum += hb;
            }
        }
        __syncthreads();
    };
    if (!keep_all) {
        need = (uint32_t)k;
        bool in_smem = false;
        uint32_t ncand = 0;
#pragma unroll 1
        for (int pass = 0; pass < 3; ++pass) {
            const int sh = pass == 0 ? 21 : (pass == 1 ? 10 : 0);
            const uint32_t nb = pass == 2 ? 1024u : 2048u;
            for (int i = tid; i < kSelBins; i += kTkThreads) h[i] = 0u;
            __syncthreads();
            if (in_smem) {   // the candidates of the threshold bucket (pass >= 1)
                for (uint32_t i = tid; i < ncand; i += kTkThreads) {
                    const uint32_t sc = cand[i];
                    if ((sc & pmask) == T) atomicAdd(&h[(sc >> sh) & (nb - 1u)], 1u);
                }
            } else {         // the segment's values in global memory
                for (uint32_t i0 = lo + tid; i0 < hi; i0 += 8u * kTkThreads) {
                    uint32_t b[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t i = i0 + (uint32_t)u * kTkThreads;
                        b[u] = i < hi ? __float_as_uint(vals[i]) : 0u;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t sc = score_bits(b[u], attn);
                        if (i0 + (uint32_t)u * kTkThreads < hi && (sc & pmask) == T)
                            atomicAdd(&h[(sc >> sh) & (nb - 1u)], 1u);
                    }
                }
            }
            __syncthreads();
            find_bin(nb);
            T |= sh_bin << sh;
            pmask |= (nb - 1u) << sh;
            need = sh_need;
            const uint32_t bcnt = sh_cnt;
            if (bcnt == need) break;   // the whole bucket is kept: no tie split below it
            if (pass == 0 && bcnt <= kTkCand) {
                // gather the bucket's scores into shared memory; the later digits run there
                __syncthreads();   // every thread has read sh_cnt before it is reused as the cursor
                if (tid == 0) sh_cnt = 0;
                __syncthreads();
                // warp-uniform trip count (the ballots below need every lane)
                for (uint32_t w0 = lo + (uint32_t)(tid - lane); w0 < hi; w0 += 8u * kTkThreads) {
                    const uint32_t i0 = w0 + (uint32_t)lane;
                    uint32_t b[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t i = i0 + (uint32_t)u * kTkThreads;
                        b[u] = i < hi ? __float_as_uint(vals[i]) : 0u;
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const uint32_t sc = score_bits(b[u], attn);
                        const bool c = i0 + (uint32_t)u * kTkThreads < hi && (sc & pmask) == T;
                        const unsigned mk = __ballot_sync(kFull, c);
                        uint32_t slot = 0;
                        if (lane == 0 && mk) slot = atomicAdd(&sh_cnt, (uint32_t)__popc(mk));
                        slot = __shfl_sync(kFull, slot, 0);
                        if (c) cand[slot + __popc(mk & ((1u << lane) - 1u))] = sc;
                    }
                }
                __syncthreads();
                ncand = sh_cnt;
                in_smem = true;
            }
        }
    }
    // ordered compaction
    const uint64_t obase = seg_off[s];
    uint32_t tie_carry = 0;
    uint64_t out_carry = 0;
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll 1
    for (uint32_t t0 = lo; t0 < hi; t0 += kTkTile) {
        const uint32_t w0 = t0 + (uint32_t)warp * (32u * kTkG);
        uint32_t bits[kTkG];
        unsigned kb[kTkG], tb[kTkG];
        uint32_t ntie = 0;
        // values and keys together (one round trip; the keys' sectors are fetched anyway at
        // these kept fractions)
        uint64_t kk[kTkG];
#pragma unroll
        for (int g = 0; g < kTkG; ++g) {
            const uint32_t i = w0 + 32u * g + lane;
            bits[g] = i < hi ? __float_as_uint(vals[i]) : 0u;
            kk[g] = i < hi ? keys[i] : 0ull;
        }
#pragma unroll
        for (int g = 0; g < kTkG; ++g) {
            const uint32_t i = w0 + 32u * g + lane;
            const bool in = i < hi;
            const uint32_t sc = score_bits(bits[g], attn) & pmask;
            const bool keep = in && (keep_all || sc > T), tie = in && !keep_all && sc == T;
            kb[g] = __ballot_sync(kFull, keep);
            tb[g] = __ballot_sync(kFull, tie);
            ntie += (uint32_t)__popc(tb[g]);
        }
        if (!keep_all) {   // block-uniform: rank the ties in key order, keep the first `need`
            if (lane == 0) wt[warp] = ntie;
            __syncthreads();
            if (warp == 0) {
                const uint32_t v = lane < kTkWarps ? wt[lane] : 0u;
                const uint32_t inc = warp_incl_scan(v);
                if (lane < kTkWarps) wt[lane] = inc - v;
                if (lane == 31) wt[kTkWarps] = inc;
            }
            __syncthreads();
            uint32_t r = tie_carry + wt[warp];
#pragma unroll
            for (int g = 0; g < kTkG; ++g) {
                const bool tie = (tb[g] >> lane) & 1u;
                const bool take = tie && r + (uint32_t)__popc(tb[g] & lt) < need;
                kb[g] |= __ballot_sync(kFull, take);
                r += (uint32_t)__popc(tb[g]);
            }
            tie_carry += wt[kTkWarps];
        }
        uint32_t nk = 0;
#pragma unroll
        for (int g = 0; g < kTkG; ++g) nk += (uint32_t)__popc(kb[g]);
        if (lane == 0) wk[warp] = nk;
        __syncthreads();
        if (warp == 0) {
            const uint32_t v = lane < kTkWarps ? wk[lane] : 0u;
            const uint32_t inc = warp_incl_scan(v);
            if (lane < kTkWarps) wk[lane] = inc - v;
            if (lane == 31) wk[kTkWarps] = inc;
        }
        __syncthreads();
        uint64_t pos = obase + out_carry + wk[warp];
#pragma unroll
        for (int g = 0; g < kTkG; ++g) {
            if ((kb[g] >> lane) & 1u) {
                const uint32_t i = w0 + 32u * g + lane;
                const uint64_t o = pos + (uint32_t)__popc(kb[g] & lt);
                ok.put(o, kk[g]);
                ov[o] = __uint_as_float(bits[g]);
                if (osrc) osrc[o] = (int64_t)i;
            }
            pos += (uint32_t)__popc(kb[g]);
        }
        out_carry += wk[kTkWarps];
        __syncthreads();   // wt / wk are rewritten by the next tile
    }
}

cudaError_t launch_topk(Keys keys, const float* vals, const uint32_t* row_ptr, int64_t R, int64_t nseg,
                        int attn, int64_t k, uint64_t* seg_off, KeysOut out_keys, float* out_vals, int64_t* out_src,
                        int64_t* out_nnz, cudaStream_t s) {
    if (nseg == 0) return cudaMemsetAsync(out_nnz, 0, sizeof(int64_t), s);
    { SPC_PHASE("topk_offsets", s, 1); topk_offsets_kernel<<<1, 1024, 0, s>>>(row_ptr, R, nseg, k, seg_off, out_nnz); }
    {
        SPC_PHASE("topk_select", s, 1);
        topk_seg_kernel<<<(unsigned)nseg, kTkThreads, 0, s>>>(keys, vals, row_ptr, R, attn, k, seg_off, out_keys,
                                                              out_vals, out_src);
    }
    return cudaGetLastError();
}

}  // namespace spc

// Attention = k-selection per output channel (§3.2) + compaction + key
// compression + write.
//
// Exact radix select on order-preserving u32 scores (|y| bits for variant (ii), sign-folded y
// for variant (i)): three digit passes (11, 11, 10 bits) find the k-th largest score T and the
// number `need` of entries equal to T that are kept (reading R7: ties go to smaller keys).
// Then an ordered compaction keeps score > T and the first `need` entries with score == T in
// key order. The same kernels serve the fused convolution (source = the dense pre-attention
// buffer with absent markers) and the standalone attention layer (source = a COO map).
// Chunks of 4096 elements never straddle segments, so per-segment ranks are two-level scans.
#include "spc_internal.cuh"
#include "block_scan.cuh"

namespace spc {

constexpr int kSelThreads = 256;
constexpr int kSelItems = kSelChunk / kSelThreads;   // 16

template <int KIND>
__device__ __forceinline__ void chunk_range(const SelSrc& S, int64_t s, int64_t c, int64_t& lo, int64_t& hi) {
    if (KIND == 0) {
        lo = c * kSelChunk;
        hi = min(S.V, lo + kSelChunk);
    } else {
        const int64_t o0 = S.row_ptr[s * S.R], o1 = S.row_ptr[(s + 1) * S.R];
        lo = o0 + c * kSelChunk;
        hi = min(o1, lo + kSelChunk);
    }
}

// element i of segment s (i absolute for COO, within-segment for dense)
template <int KIND>
__device__ __forceinline__ uint32_t elem_bits(const SelSrc& S, int64_t s, int64_t i) {
    if (KIND == 0) return __float_as_uint(S.pre[s * S.V + i]);
    return __float_as_uint(S.vals[i]);
}
template <int KIND>
__device__ __forceinline__ bool present(uint32_t bits) {
    return KIND == 0 ? bits != kAbsent : true;
}

template <int KIND>
__global__ void sel_init_kernel(SelSrc S, int64_t k, SelState* st, uint32_t* hist) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S.nseg; s += (int64_t)gridDim.x * blockDim.x) {
        int64_t n;
        if (KIND == 0) n = (int64_t)S.seg_count[s];
        else n = (int64_t)S.row_ptr[(s + 1) * S.R] - (int64_t)S.row_ptr[s * S.R];
        SelState x{};
        if (S.attn == SPC_ATTN_NONE || n <= k) {
            x.keep_all = 1;
            x.kept = n;
            x.need = 0;
        } else {
            x.keep_all = 0;
            x.kept = k;
            x.need = k;
        }
        x.prefix = 0;
        x.pmask = 0;
        st[s] = x;
    }
}

template <int KIND>
__global__ void __launch_bounds__(kSelThreads) sel_hist_kernel(SelSrc S, const SelState* __restrict__ st,
                                                               uint32_t* __restrict__ hist, int sh, int nbits) {
    const int64_t s = (int64_t)blockIdx.x / S.nchunk, c = (int64_t)blockIdx.x % S.nchunk;
    const SelState x = st[s];
    if (x.keep_all) return;
    int64_t lo, hi;
    chunk_range<KIND>(S, s, c, lo, hi);
    if (lo >= hi) return;
    __shared__ uint32_t h[kSelBins];
    for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint32_t dmask = (1u << nbits) - 1u;
#pragma unroll 4
    for (int u = 0; u < kSelItems; ++u) {
        const int64_t i = lo + (int64_t)u * kSelThreads + threadIdx.x;
        if (i < hi) {
            const uint32_t bits = elem_bits<KIND>(S, s, i);
            if (present<KIND>(bits)) {
                const uint32_t sc = score_bits(bits, S.attn);
                if ((sc & x.pmask) == x.prefix) atomicAdd(&h[(sc >> sh) & dmask], 1u);
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= (int)dmask; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[s * kSelBins + i], h[i]);
}

// Per segment: walk the bins from the top until the running count reaches `need`.
__global__ void __launch_bounds__(kSelThreads) sel_find_kernel(SelState* st, uint32_t* hist, int sh, int nbits) {
    const int64_t s = blockIdx.x;
    __shared__ uint64_t sm[33];
    __shared__ int found;
    SelState x = st[s];
    if (x.keep_all) return;
    const int nb = 1 << nbits;
    const int per = nb / kSelThreads;   // 8 or 4 bins per thread
    uint32_t* h = hist + s * kSelBins;
    // thread t owns bins [nb-1-t*per-(per-1), nb-1-t*per], scanned from the top
    uint64_t local = 0;
    for (int q = 0; q < per; ++q) local += h[nb - 1 - threadIdx.x * per - q];
    uint64_t tot;
    const uint64_t before = block_excl_scan(local, sm, &tot);
    if (threadIdx.x == 0) found = 0;
    __syncthreads();
    const uint64_t need = (uint64_t)x.need;
    if (before < need && before + local >= need) {
        uint64_t cum = before;
        for (int q = 0; q < per; ++q) {
            const int bin = nb - 1 - threadIdx.x * per - q;
            const uint64_t hb = h[bin];
            if (cum + hb >= need) {
                x.need = (int64_t)(need - cum);
                x.prefix |= (uint32_t)bin << sh;
                x.pmask |= (uint32_t)(nb - 1) << sh;
                st[s] = x;
                found = 1;
                break;
            }
            cum += hb;
        }
    }
    __syncthreads();
    // reset this segment's histogram for the next pass
    for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) h[i] = 0;
}

template <int KIND>
__global__ void __launch_bounds__(kSelThreads) sel_count_kernel(SelSrc S, const SelState* __restrict__ st,
                                                                ChunkRec* __restrict__ rec) {
    const int64_t s = (int64_t)blockIdx.x / S.nchunk, c = (int64_t)blockIdx.x % S.nchunk;
    const SelState x = st[s];
    int64_t lo, hi;
    chunk_range<KIND>(S, s, c, lo, hi);
    uint32_t gt = 0, eq = 0;
    for (int u = 0; u < kSelItems; ++u) {
        const int64_t i = lo + (int64_t)u * kSelThreads + threadIdx.x;
        if (i < hi) {
            const uint32_t bits = elem_bits<KIND>(S, s, i);
            if (present<KIND>(bits)) {
                if (x.keep_all) ++gt;
                else {
                    const uint32_t sc = score_bits(bits, S.attn);
                    gt += sc > x.prefix;
                    eq += sc == x.prefix;
                }
            }
        }
    }
    __shared__ uint32_t sm[33];
    const uint32_t g = block_sum(gt, sm);
    const uint32_t e = block_sum(eq, sm);
    if (threadIdx.x == 0) {
        ChunkRec r{};
        r.gt = g;
        r.eq = e;
        rec[s * S.nchunk + c] = r;
    }
}

// Per segment: ordered prefix over chunks of ties and kept entries.
__global__ void sel_chunk_scan_kernel(int64_t nchunk, const SelState* __restrict__ st, ChunkRec* __restrict__ rec,
                                      uint64_t* __restrict__ seg_kept) {
    const int64_t s = blockIdx.x;
    const SelState x = st[s];
    __shared__ uint64_t sm[33];
    uint64_t tie_carry = 0, keep_carry = 0;
    for (int64_t base = 0; base < nchunk; base += blockDim.x) {
        const int64_t c = base + threadIdx.x;
        ChunkRec r{};
        if (c < nchunk) r = rec[s * nchunk + c];
        uint64_t tt;
        const uint64_t tb = block_excl_scan((uint64_t)r.eq, sm, &tt) + tie_carry;
        uint64_t keep = r.gt;
        if (!x.keep_all) {
            const int64_t rem = x.need - (int64_t)tb;
            keep += rem <= 0 ? 0 : (rem >= (int64_t)r.eq ? r.eq : (uint64_t)rem);
        }
        uint64_t kt;
        const uint64_t kb = block_excl_scan(keep, sm, &kt) + keep_carry;
        if (c < nchunk) {
            r.tie_before = tb;
            r.out_off = kb;
            rec[s * nchunk + c] = r;
        }
        tie_carry += tt;
        keep_carry += kt;
    }
    if (threadIdx.x == 0) seg_kept[s] = keep_carry;
}

__global__ void seg_scan_kernel(uint64_t* seg, int64_t nseg, int64_t* total) {
    __shared__ uint64_t sm[33];
    uint64_t carry = 0;
    for (int64_t base = 0; base < nseg; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const uint64_t v = i < nseg ? seg[i] : 0;
        uint64_t t;
        const uint64_t ex = block_excl_scan(v, sm, &t);
        if (i < nseg) seg[i] = carry + ex;
        carry += t;
    }
    if (threadIdx.x == 0 && total) *total = (int64_t)carry;
}

template <int KIND>
__global__ void __launch_bounds__(kSelThreads) sel_write_kernel(SelSrc S, const SelState* __restrict__ st,
                                                                const ChunkRec* __restrict__ rec,
                                                                const uint64_t* __restrict__ seg_off,
                                                                uint64_t* __restrict__ out_keys,
                                                                float* __restrict__ out_vals,
                                                                int64_t* __restrict__ out_src) {
    const int64_t s = (int64_t)blockIdx.x / S.nchunk, c = (int64_t)blockIdx.x % S.nchunk;
    int64_t lo, hi;
    chunk_range<KIND>(S, s, c, lo, hi);
    if (lo >= hi) return;
    const SelState x = st[s];
    const ChunkRec r = rec[s * S.nchunk + c];
    const int64_t my = lo + (int64_t)threadIdx.x * kSelItems;
    uint32_t bits[kSelItems];
    uint8_t cls[kSelItems];   // 0 drop, 1 keep, 2 tie
    uint32_t neq = 0;
#pragma unroll
    for (int u = 0; u < kSelItems; ++u) {
        const int64_t i = my + u;
        cls[u] = 0;
        bits[u] = 0;
        if (i < hi) {
            bits[u] = elem_bits<KIND>(S, s, i);
            if (present<KIND>(bits[u])) {
                if (x.keep_all) cls[u] = 1;
                else {
                    const uint32_t sc = score_bits(bits[u], S.attn);
                    cls[u] = sc > x.prefix ? 1 : (sc == x.prefix ? 2 : 0);
                    neq += cls[u] == 2;
                }
            }
        }
    }
    __shared__ uint32_t sm[33];
    uint32_t t_eq;
    uint64_t tie = r.tie_before + block_excl_scan(neq, sm, &t_eq);
    uint32_t nkeep = 0;
#pragma unroll
    for (int u = 0; u < kSelItems; ++u) {
        if (cls[u] == 2) {
            cls[u] = ((int64_t)tie < x.need) ? 1 : 0;
            ++tie;
        }
        nkeep += cls[u] == 1;
    }
    uint32_t t_keep;
    uint64_t pos = seg_off[s] + r.out_off + block_excl_scan(nkeep, sm, &t_keep);
#pragma unroll
    for (int u = 0; u < kSelItems; ++u) {
        if (cls[u] == 1) {
            const int64_t i = my + u;
            out_keys[pos] = KIND == 0 ? (uint64_t)(s * S.V + i) : S.keys[i];
            out_vals[pos] = __uint_as_float(bits[u]);
            if (out_src) out_src[pos] = KIND == 0 ? -1 : i;
            ++pos;
        }
    }
}

template <int KIND>
static cudaError_t run_select(const SelSrc& S, int64_t k, SelState* st, uint32_t* hist, ChunkRec* rec,
                              uint64_t* seg_off, uint64_t* out_keys, float* out_vals, int64_t* out_src,
                              int64_t* out_nnz, cudaStream_t s) {
    if (S.nseg == 0) return cudaMemsetAsync(out_nnz, 0, sizeof(int64_t), s);
    const unsigned gs = (unsigned)((S.nseg + 255) / 256);
    { SPC_PHASE("sel_init", s, 1); sel_init_kernel<KIND><<<gs, 256, 0, s>>>(S, k, st, hist); }
    const unsigned grid = (unsigned)(S.nchunk * S.nseg);
    if (S.attn != SPC_ATTN_NONE) {
        cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(uint32_t) * kSelBins * (size_t)S.nseg, s);
        if (e != cudaSuccess) return e;
        const int shs[3] = {21, 10, 0};
        const int nbs[3] = {11, 11, 10};
        for (int p = 0; p < 3; ++p) {
            { SPC_PHASE("sel_hist", s, 1); sel_hist_kernel<KIND><<<grid, kSelThreads, 0, s>>>(S, st, hist, shs[p], nbs[p]); }
            { SPC_PHASE("sel_find", s, 1); sel_find_kernel<<<(unsigned)S.nseg, kSelThreads, 0, s>>>(st, hist, shs[p], nbs[p]); }
        }
    }
    { SPC_PHASE("sel_count", s, 1); sel_count_kernel<KIND><<<grid, kSelThreads, 0, s>>>(S, st, rec); }
    { SPC_PHASE("sel_chunk_scan", s, 1); sel_chunk_scan_kernel<<<(unsigned)S.nseg, 1024, 0, s>>>(S.nchunk, st, rec, seg_off); }
    { SPC_PHASE("seg_scan", s, 1); seg_scan_kernel<<<1, 1024, 0, s>>>(seg_off, S.nseg, out_nnz); }
    { SPC_PHASE("sel_write", s, 1); sel_write_kernel<KIND><<<grid, kSelThreads, 0, s>>>(S, st, rec, seg_off, out_keys, out_vals, out_src); }
    return cudaGetLastError();
}

cudaError_t launch_select(const SelSrc& src, int64_t k, SelState* st, uint32_t* hist, ChunkRec* rec,
                          uint64_t* seg_off, uint64_t* out_keys, float* out_vals, int64_t* out_src,
                          int64_t* out_nnz, cudaStream_t s) {
    if (src.kind == 0)
        return run_select<0>(src, k, st, hist, rec, seg_off, out_keys, out_vals, out_src, out_nnz, s);
    return run_select<1>(src, k, st, hist, rec, seg_off, out_keys, out_vals, out_src, out_nnz, s);
}

}  // namespace spc

// Index structures (Alg. 1 step 1 "decompress filter and data indices"), device-wide
// scan, validation and small helpers. Internal to libspconv.
#include "spc_internal.cuh"
#include "block_scan.cuh"

#include <algorithm>

namespace spc {

// ------------------------------------------------------------------------ segment bounds
// seg_ptr[s] = first entry whose key >= s*V, s in [0, nseg]: one binary search per segment (the
// per-(b, c) bounds of a map without its full row index -- the standalone attention needs only
// these).
// One warp per bound: a 32-ary search (32 probes per step, a ballot picks the sub-range), about
// log32(n) + 1 dependent loads instead of log2(n).
__global__ void seg_bounds_kernel(Keys keys, const int64_t* nnz_dev, int64_t nbound, int64_t nseg, uint64_t V,
                                  uint32_t* __restrict__ seg_ptr) {
    const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s > nseg) return;
    const int64_t n = load_n(nnz_dev, nbound);
    const uint64_t want = (uint64_t)s * V;
    int64_t lo = 0, hi = n;   // first i with keys[i] >= want lies in [lo, hi]
    while (hi - lo > 32) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t p = lo + (int64_t)(lane + 1) * step - 1;
        const bool below = p < hi && keys[p] < want;
        const int c = __popc(__ballot_sync(0xffffffffu, below));
        const int64_t nlo = lo + (int64_t)c * step;
        hi = min(hi, lo + (int64_t)(c + 1) * step - 1);
        lo = nlo;
    }
    const bool below = lo + lane < hi && keys[lo + lane] < want;
    const int c = __popc(__ballot_sync(0xffffffffu, below));
    if (lane == 0) seg_ptr[s] = (uint32_t)(lo + c);
}

cudaError_t launch_seg_bounds(Keys keys, const int64_t* nnz_dev, int64_t nbound, int64_t nseg, int64_t V,
                              uint32_t* seg_ptr, cudaStream_t s) {
    SPC_PHASE("seg_bounds", s, 1);
    seg_bounds_kernel<<<(unsigned)((32 * (nseg + 1) + 255) / 256), 256, 0, s>>>(keys, nnz_dev, nbound, nseg,
                                                                                 (uint64_t)V, seg_ptr);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------- row index
// row_ptr[r] = first entry whose key >= r*Z, for r in [0, total_rows]. A block computes the rows
// of its 2048 entries from coalesced key loads into shared memory; then each entry fills the gap
// of rows between its predecessor's row and its own (consecutive entries on consecutive lanes);
// long empty stretches are filled by the whole warp so they do not serialise on one thread.
// key / Z by a multiply-high with a host-computed reciprocal and one exact correction; 32-bit
// arithmetic throughout when the key space fits (batch*channels*V <= 2^32, the "Sparse 32"
// condition of Table 1), 64-bit otherwise.
constexpr int kRiItems = 8;

__device__ __forceinline__ int64_t row_of(uint64_t key, uint64_t Z, uint64_t magic) {
    uint64_t q = __umul64hi(key, magic);   // floor(key / Z) or one less
    if ((q + 1) * Z <= key) ++q;
    return (int64_t)q;
}
__device__ __forceinline__ int32_t row_of(uint32_t key, uint32_t Z, uint32_t magic) {
    uint32_t q = __umulhi(key, magic);     // floor(key / Z) or one less
    if ((uint64_t)(q + 1) * Z <= key) ++q;
    return (int32_t)q;
}

template <typename K, typename I, bool K32>   // key word, row / entry index type, 32-bit key storage
__global__ void __launch_bounds__(256) row_index_kernel(K Z, K magic, Keys keys,
                                                        const int64_t* nnz_dev, int64_t nbound,
                                                        uint32_t* __restrict__ row_ptr, I total_rows,
                                                        const float* __restrict__ vals, int* __restrict__ guard) {
    constexpr int kB = 256 * kRiItems;   // entries per block
    __shared__ I srow[kB + 1];           // srow[1 + t] = row of entry b0 + t; srow[0] = row of b0 - 1
    const I n = (I)load_n(nnz_dev, nbound);
    const I b0 = (I)blockIdx.x * kB;
    if (b0 > n) return;
    const int lane = threadIdx.x & 31;
    // rows of the block's entries, computed from coalesced key loads
    bool tiny = false;   // the forward's value guard (value_guard_kernel), fused when vals != null
#pragma unroll
    for (int q = 0; q < kRiItems; ++q) {
        const int t = q * 256 + threadIdx.x;
        const I i = b0 + t;
        srow[1 + t] = i < n ? (I)row_of((K)keys.template at<K32>(i), Z, magic) : total_rows;
        if (vals && i < n) {
            const float v = vals[i];
            tiny |= !(fabsf(v) >= 0x1p-50f) && !isnan(v);
        }
    }
    if (threadIdx.x == 0) srow[0] = b0 == 0 ? (I)-1 : (I)row_of((K)keys.template at<K32>(b0 - 1), Z, magic);
    if (__syncthreads_or(tiny) && threadIdx.x == 0) *guard = 1;
    // entry i (and the sentinel i = n) fills the rows between its predecessor's row and its own
#pragma unroll
    for (int q = 0; q < kRiItems; ++q) {
        const int t = q * 256 + threadIdx.x;
        const I i = b0 + t;
        I lo = 0, hi = -1;
        if (i <= n) {
            lo = srow[t] + 1;
            const I r = srow[t + 1];
            hi = (i < n && r < total_rows) ? r : total_rows;
        }
        const bool longgap = hi - lo >= 16;
        if (!longgap)
            for (I r = lo; r <= hi; ++r) row_ptr[r] = (uint32_t)i;
        unsigned m = __ballot_sync(kFull, longgap);
        while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const I l = __shfl_sync(kFull, lo, src);
            const I h = __shfl_sync(kFull, hi, src);
            const I v = __shfl_sync(kFull, i, src);
            for (I r = l + lane; r <= h; r += 32) row_ptr[r] = (uint32_t)v;
        }
    }
}

cudaError_t launch_row_index(const Geo& g, Keys keys, const int64_t* nnz_dev, int64_t nbound,
                             uint32_t* row_ptr, cudaStream_t s, const float* vals, int* guard) {
    const int64_t total_rows = g.B * g.C * g.R;
    const int bs = 256;
    const int64_t grid = (nbound + 1 + (int64_t)bs * kRiItems - 1) / ((int64_t)bs * kRiItems);
    const double space = (double)g.B * (double)g.C * (double)g.V;
    SPC_PHASE("row_index", s, 1);
    if (space <= 4294967296.0 && nbound < (1ll << 30) && total_rows < (1ll << 30)) {
        const uint32_t Z = (uint32_t)g.Z;
        const uint32_t magic = Z == 1 ? ~0u : ~0u / Z;
        if (keys.k32)
            row_index_kernel<uint32_t, int32_t, true><<<(unsigned)grid, bs, 0, s>>>(Z, magic, keys, nnz_dev, nbound,
                                                                                  row_ptr, (int32_t)total_rows, vals, guard);
        else
            row_index_kernel<uint32_t, int32_t, false><<<(unsigned)grid, bs, 0, s>>>(Z, magic, keys, nnz_dev, nbound,
                                                                                   row_ptr, (int32_t)total_rows, vals, guard);
    } else {
        const uint64_t Z = (uint64_t)g.Z;
        const uint64_t magic = Z == 1 ? ~0ull : ~0ull / Z;   // floor((2^64 - 1) / Z)
        row_index_kernel<uint64_t, int64_t, false><<<(unsigned)grid, bs, 0, s>>>(Z, magic, keys, nnz_dev, nbound, row_ptr,
                                                                                   total_rows, vals, guard);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------------- filter table
// Both tables re-lay the key-sorted filter, whose groups (of the target order) are contiguous key
// runs: (1) grid-wide, entry j opens its group's run when its predecessor is in another group and
// closes it likewise; (2) one block clamps the runs and scans their lengths into offsets; (3)
// grid-wide, every entry moves to its slot. K: uint32_t when every filter key is below 2^32
// (c_out * c_in * prod(ksize), always in practice): the key arithmetic avoids emulated 64-bit
// divisions.
template <typename K>
struct GrpBwd {   // (oc, ic) of a key, ic-major target order q = oc*c_in + ic (run index)
    KGeo kg;
    __device__ int operator()(const uint64_t* wk, int64_t j) const { return (int)((K)wk[j] / (K)kg.KV); }
};
template <typename K>
struct GrpFwd {   // q = (ic*KXY + dxdy)*c_out + oc
    KGeo kg;
    int c_in, c_out, KXY;
    __device__ int operator()(const uint64_t* wk, int64_t j) const {
        const K k = (K)wk[j];
        const K pq = k / (K)kg.KV;
        const int oc = (int)(pq / (K)c_in), ic = (int)(pq - (K)oc * (K)c_in);
        const int dxdy = (int)((k - pq * (K)kg.KV) / (K)kg.kz);
        return (ic * KXY + dxdy) * c_out + oc;
    }
};

// run_start / run_len zeroed by the caller; run_len[q] receives the run's end
template <typename G>
__global__ void filter_runs_kernel(const uint64_t* __restrict__ wk, int64_t nw, int nq, G grp,
                                   int* __restrict__ run_start, int* __restrict__ run_len) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nw; j += (int64_t)gridDim.x * blockDim.x) {
        const int q = grp(wk, j);
        if (q < 0 || q >= nq) continue;   // out-of-range filter key (rejected under SPC_VALIDATE)
        if (j == 0 || grp(wk, j - 1) != q) run_start[q] = (int)j;
        if (j + 1 == nw || grp(wk, j + 1) != q) run_len[q] = (int)j + 1;
    }
}

// (unsorted or duplicated keys break the runs: clamped so that no write leaves the tables)
__device__ __forceinline__ int run_len_of(const int* run_start, const int* run_len, int q, int64_t nw) {
    return max(0, min(run_len[q] - run_start[q], (int)nw - run_start[q]));
}

// backward table (ic, oc, delta): off[ic*(c_out+1) + oc] = first entry of (oc, ic)
__global__ void filter_bwd_offsets_kernel(int c_in, int c_out, int64_t nw, const int* __restrict__ run_start,
                                          int* __restrict__ run_len, int* __restrict__ off) {
    __shared__ int sm[33];
    const int npairs = c_in * c_out;
    int carry = 0;
    for (int base = 0; base < npairs; base += blockDim.x) {
        const int q = base + threadIdx.x;          // ic-major: q = ic*c_out + oc
        int len = 0, ic = 0, oc = 0;
        if (q < npairs) {
            ic = q / c_out;
            oc = q - ic * c_out;
            len = run_len_of(run_start, run_len, oc * c_in + ic, nw);
        }
        int tot;
        const int ex = block_excl_scan(len, sm, &tot);
        if (q < npairs) off[ic * (c_out + 1) + oc] = carry + ex;
        carry += tot;
    }
    __syncthreads();
    for (int ic = threadIdx.x; ic < c_in; ic += blockDim.x)
        off[ic * (c_out + 1) + c_out] = (ic + 1 < c_in) ? off[(ic + 1) * (c_out + 1)] : carry;
}

template <typename K>
__global__ void filter_bwd_scatter_kernel(KGeo kg, int c_in, int c_out, const uint64_t* __restrict__ wk,
                                          const float* __restrict__ wv, int64_t nw, int2* __restrict__ meta,
                                          float* __restrict__ val, const int* __restrict__ off,
                                          int* __restrict__ src, const int* __restrict__ run_start) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nw; j += (int64_t)gridDim.x * blockDim.x) {
        const K key = (K)wk[j];
        const int p = (int)(key / (K)kg.KV);
        const int dlin = (int)(key - (K)p * (K)kg.KV);
        if (p >= c_in * c_out) continue;   // out-of-range key (rejected under SPC_VALIDATE)
        const int oc = p / c_in, ic = p - (p / c_in) * c_in;
        const int dst = off[ic * (c_out + 1) + oc] + (int)(j - run_start[p]);
        if (dst < 0 || dst >= nw) continue;
        const int dz = dlin % kg.kz;
        const int dy = (dlin / kg.kz) % kg.ky;
        const int dx = (dlin / (kg.kz * kg.ky)) % kg.kx;
        const int dw = dlin / (kg.kz * kg.ky * kg.kx);
        meta[dst] = make_int2(pack_oc_ow(oc, dw - kg.hw), pack_off(dx - kg.hx, dy - kg.hy, dz - kg.hz));
        val[dst] = wv[j];
        src[dst] = (int)j;
    }
}

static unsigned table_grid(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 4 * num_sms())); }

// Re-lays the (oc, ic, delta)-sorted filter into ic-major order (ic, oc, delta) so that a CTA
// finds "filter(oc, ic)" of Alg. 1 for a group of oc as one contiguous range.
cudaError_t launch_filter_table(const KGeo& kg, int c_in, int c_out, const uint64_t* wkeys, const float* wvals,
                                int64_t nw, int2* meta, float* val, int* off, int* src, int* scratch, cudaStream_t s) {
    const int npairs = c_in * c_out;
    int* run_start = scratch;
    int* run_len = scratch + (size_t)npairs;
    SPC_PHASE("filter_table", s, 3);
    cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(int) * 2 * (size_t)npairs, s);
    if (e != cudaSuccess) return e;
    const bool k32 = (double)c_out * c_in * kg.KV <= 4294967295.0;
    if (k32) filter_runs_kernel<<<table_grid(nw), 256, 0, s>>>(wkeys, nw, npairs, GrpBwd<uint32_t>{kg}, run_start, run_len);
    else filter_runs_kernel<<<table_grid(nw), 256, 0, s>>>(wkeys, nw, npairs, GrpBwd<uint64_t>{kg}, run_start, run_len);
    filter_bwd_offsets_kernel<<<1, 1024, 0, s>>>(c_in, c_out, nw, run_start, run_len, off);
    if (k32)
        filter_bwd_scatter_kernel<uint32_t><<<table_grid(nw), 256, 0, s>>>(kg, c_in, c_out, wkeys, wvals, nw, meta, val, off,
                                                                            src, run_start);
    else
        filter_bwd_scatter_kernel<uint64_t><<<table_grid(nw), 256, 0, s>>>(kg, c_in, c_out, wkeys, wvals, nw, meta, val, off,
                                                                            src, run_start);
    return cudaGetLastError();
}

// Second order of the filter for the forward kernel: (ic, (dx,dy), oc, dz). For a fixed input
// channel and in-plane offset the weights of a group of output channels are then one
// contiguous range. meta2[j] = {oc, oz}, off2[(ic*KXY + dxdy)*(c_out+1) + oc] = first entry.
// scratch: 2 * c_in*KXY*c_out ints.
__global__ void filter_fwd_offsets_kernel(int nq, int c_out, int64_t nw, const int* __restrict__ run_start,
                                          const int* __restrict__ run_len, int* __restrict__ off2) {
    __shared__ int sm[33];
    const int ng = nq / c_out;
    int carry = 0;
    for (int base = 0; base < nq; base += blockDim.x) {
        const int q = base + threadIdx.x;
        const int len = q < nq ? run_len_of(run_start, run_len, q, nw) : 0;
        int tot;
        const int ex = block_excl_scan(len, sm, &tot);
        if (q < nq) off2[(q / c_out) * (c_out + 1) + q % c_out] = carry + ex;
        carry += tot;
    }
    __syncthreads();
    for (int g = threadIdx.x; g < ng; g += blockDim.x)
        off2[g * (c_out + 1) + c_out] = (g + 1 < ng) ? off2[(g + 1) * (c_out + 1)] : carry;
}

template <typename K>
__global__ void filter_fwd_scatter_kernel(KGeo kg, int nq, int c_out, const uint64_t* __restrict__ wk,
                                          const float* __restrict__ wv, int64_t nw, int2* __restrict__ meta2,
                                          float* __restrict__ val2, const int* __restrict__ off2,
                                          const int* __restrict__ run_start, const int* __restrict__ run_len) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nq; q += gridDim.x * blockDim.x) {
        const int oc = q % c_out, g = q / c_out;
        const int dst = off2[g * (c_out + 1) + oc];
        const int n = run_len_of(run_start, run_len, q, nw);
        for (int i = 0; i < n && dst + i < nw; ++i) {
            const int j = run_start[q] + i;
            const int dz = (int)((K)wk[j] % (K)kg.kz);
            meta2[dst + i] = make_int2(oc, dz - kg.hz);
            val2[dst + i] = wv[j];
        }
    }
}

cudaError_t launch_filter_table_fwd(const KGeo& kg, int c_in, int c_out, const uint64_t* wkeys, const float* wvals,
                                    int64_t nw, int2* meta2, float* val2, int* off2, int* scratch, cudaStream_t s) {
    const int KXY = kg.kw * kg.kx * kg.ky;
    const int nq = c_in * KXY * c_out;
    int* run_start = scratch;
    int* run_len = scratch + (size_t)nq;
    SPC_PHASE("filter_table", s, 3);
    cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(int) * 2 * (size_t)nq, s);
    if (e != cudaSuccess) return e;
    const bool k32 = (double)c_out * c_in * kg.KV <= 4294967295.0;
    if (k32)
        filter_runs_kernel<<<table_grid(nw), 256, 0, s>>>(wkeys, nw, nq, GrpFwd<uint32_t>{kg, c_in, c_out, KXY}, run_start,
                                                          run_len);
    else
        filter_runs_kernel<<<table_grid(nw), 256, 0, s>>>(wkeys, nw, nq, GrpFwd<uint64_t>{kg, c_in, c_out, KXY}, run_start,
                                                          run_len);
    filter_fwd_offsets_kernel<<<1, 1024, 0, s>>>(nq, c_out, nw, run_start, run_len, off2);
    if (k32)
        filter_fwd_scatter_kernel<uint32_t><<<table_grid(nq), 256, 0, s>>>(kg, nq, c_out, wkeys, wvals, nw, meta2, val2,
                                                                            off2, run_start, run_len);
    else
        filter_fwd_scatter_kernel<uint64_t><<<table_grid(nq), 256, 0, s>>>(kg, nq, c_out, wkeys, wvals, nw, meta2, val2,
                                                                            off2, run_start, run_len);
    return cudaGetLastError();
}

// --------------------------------------------------------------------- device-wide scan
constexpr int kScanBlock = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanBlock * kScanItems;

size_t scan_tmp_words(int64_t n) { return (size_t)((n + kScanTile - 1) / kScanTile) + 2; }

__global__ void scan_reduce_kernel(const uint32_t* __restrict__ in, int64_t n, uint64_t* __restrict__ sums) {
    __shared__ uint64_t sm[33];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint64_t acc = 0;
    for (int t = 0; t < kScanItems; ++t) {
        const int64_t i = base + (int64_t)t * kScanBlock + threadIdx.x;
        if (i < n) acc += in[i];
    }
    const uint64_t tot = block_sum(acc, sm);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void scan_sums_kernel(uint64_t* sums, int64_t nb, int64_t* total) {
    __shared__ uint64_t sm[33];
    uint64_t carry = 0;
    for (int64_t base = 0; base < nb; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        const uint64_t v = i < nb ? sums[i] : 0;
        uint64_t tot;
        const uint64_t ex = block_excl_scan(v, sm, &tot);
        if (i < nb) sums[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0 && total) *total = (int64_t)carry;
}

__global__ void scan_down_kernel(const uint32_t* __restrict__ in, int64_t n, const uint64_t* __restrict__ sums,
                                 uint64_t* __restrict__ out, int64_t* __restrict__ total = nullptr) {
    __shared__ uint64_t sm[33];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint64_t acc = 0;
#pragma unroll
    for (int t = 0; t < kScanItems; ++t) {
        const int64_t i = base + t;
        v[t] = i < n ? in[i] : 0u;
        acc += v[t];
    }
    uint64_t tot;
    uint64_t ex = block_excl_scan(acc, sm, &tot) + (sums ? sums[blockIdx.x] : 0ull);
    if (total && threadIdx.x == 0) *total = (int64_t)tot;   // single-tile form
#pragma unroll
    for (int t = 0; t < kScanItems; ++t) {
        const int64_t i = base + t;
        if (i < n) out[i] = ex;
        ex += v[t];
    }
}

cudaError_t launch_scan_u32(const uint32_t* in, uint64_t* out, int64_t n, int64_t* total, uint64_t* tmp,
                            cudaStream_t s) {
    const int64_t nb = (n + kScanTile - 1) / kScanTile;
    if (nb == 1) {   // one tile: a single launch (latency-bound small layers)
        SPC_PHASE("scan_down", s, 1);
        scan_down_kernel<<<1, kScanBlock, 0, s>>>(in, n, nullptr, out, total);
        return cudaGetLastError();
    }
    if (nb > 0) { SPC_PHASE("scan_reduce", s, 1); scan_reduce_kernel<<<(unsigned)nb, kScanBlock, 0, s>>>(in, n, tmp); }
    { SPC_PHASE("scan_sums", s, 1); scan_sums_kernel<<<1, 1024, 0, s>>>(tmp, nb, total); }
    if (nb > 0) { SPC_PHASE("scan_down", s, 1); scan_down_kernel<<<(unsigned)nb, kScanBlock, 0, s>>>(in, n, tmp, out); }
    return cudaGetLastError();
}

// --------------------------------------------------------------------------- validation
__global__ void validate_kernel(Keys keys, const int64_t* nnz_dev, int64_t nbound,
                                uint64_t limit, int* flag) {
    const int64_t n = load_n(nnz_dev, nbound);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        if (k >= limit || (i > 0 && keys[i - 1] >= k)) atomicOr(flag, 1);
    }
}

cudaError_t launch_validate(Keys keys, const int64_t* nnz_dev, int64_t nbound, uint64_t limit,
                            int* flag, cudaStream_t s) {
    { SPC_PHASE("validate", s, 1); validate_kernel<<<592, 256, 0, s>>>(keys, nnz_dev, nbound, limit, flag); }
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------ helpers
__global__ void f64_to_f32_kernel(const double* __restrict__ a, float* __restrict__ b, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b[i] = (float)a[i];
}

// two ranges in one launch (the backward's dw and dbias)
__global__ void f64_to_f32_2_kernel(const double* __restrict__ a, float* __restrict__ b, int64_t n,
                                    const double* __restrict__ a2, float* __restrict__ b2, int64_t n2) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n + n2; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n) b[i] = (float)a[i];
        else b2[i - n] = (float)a2[i - n];
    }
}

cudaError_t launch_f64_to_f32_2(const double* a, float* b, int64_t n, const double* a2, float* b2, int64_t n2,
                                cudaStream_t s) {
    if (n + n2 <= 0) return cudaSuccess;
    int64_t grid = (n + n2 + 255) / 256;
    if (grid > 1184) grid = 1184;
    { SPC_PHASE("f64_to_f32", s, 1); f64_to_f32_2_kernel<<<(unsigned)grid, 256, 0, s>>>(a, b, n, a2, b2, n2); }
    return cudaGetLastError();
}

cudaError_t launch_f64_to_f32(const double* a, float* b, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int64_t grid = (n + 255) / 256;
    if (grid > 1184) grid = 1184;
    { SPC_PHASE("f64_to_f32", s, 1); f64_to_f32_kernel<<<(unsigned)grid, 256, 0, s>>>(a, b, n); }
    return cudaGetLastError();
}

// Eq. (5): the gradient passes where the forward layer kept an entry.
__global__ void scatter_grad_kernel(const int64_t* __restrict__ src, const float* __restrict__ dy, int64_t nbound,
                                    const int64_t* n_dev, float* __restrict__ dx, int64_t n_in) {
    const int64_t n = load_n(n_dev, nbound);
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = src[t];
        if (i >= 0 && i < n_in) dx[i] = dy[t];
    }
}

cudaError_t launch_scatter_grad(const int64_t* src, const float* dy, int64_t n_out_bound, const int64_t* n_out_dev,
                                float* dx, int64_t n_in, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(dx, 0, sizeof(float) * (size_t)n_in, s);
    if (e != cudaSuccess) return e;
    if (n_out_bound <= 0) return cudaSuccess;
    int64_t grid = (n_out_bound + 255) / 256;
    if (grid > num_sms() * 16) grid = num_sms() * 16;
    { SPC_PHASE("scatter_grad", s, 1); scatter_grad_kernel<<<(unsigned)grid, 256, 0, s>>>(src, dy, n_out_bound, n_out_dev, dx, n_in); }
    return cudaGetLastError();
}

// The same for a strictly increasing src (ReLU and attention_topk emit their sources in key
// order): every dx element is written exactly once, no zero fill first. CTA c owns the sources
// t in [c*T, (c+1)*T) and the dx range [a, b) from just after its predecessor's last index to its
// own last index (the CTA holding the end sentinel t = n: to n_in). When the range fits shared
// memory it is assembled there (zeros, then dy at the sources) and streamed out with 16-byte
// coalesced stores; otherwise thread t writes dy[t] and zeroes the gap after its predecessor
// (gaps of 64 or more by the whole warp).
// sources per CTA: T = 256 * items, items in {1, 2, 4, 8} chosen on the host so that small maps
// still spread over the SMs
constexpr int kSgCap = 8192;            // dx elements assembled in shared memory (32 KB)

template <int kSgT>
__global__ void __launch_bounds__(256) scatter_grad_sorted_kernel(const int64_t* __restrict__ src,
                                                                  const float* __restrict__ dy, int64_t nbound,
                                                                  const int64_t* n_dev, float* __restrict__ dx,
                                                                  int64_t n_in) {
    __shared__ __align__(16) float buf[kSgCap];
    const int64_t n = load_n(n_dev, nbound);
    const int64_t t0 = (int64_t)blockIdx.x * kSgT;
    if (t0 > n) return;
    const int64_t t1 = min(t0 + (int64_t)kSgT, n);   // sources [t0, t1); the sentinel when t1 == n
    const bool last = t0 + kSgT >= n;                   // this CTA covers the tail up to n_in
    auto clampi = [&](int64_t v) { return v < 0 ? (int64_t)0 : (v > n_in ? n_in : v); };
    const int64_t a = t0 == 0 ? 0 : clampi(src[t0 - 1] + 1);
    const int64_t b = last ? n_in : clampi(src[t1 - 1] + 1);
    const int64_t len = b > a ? b - a : 0;
    if (len <= kSgCap) {
        float4* b4 = reinterpret_cast<float4*>(buf);
        for (int i = threadIdx.x; i < (int)((len + 3) >> 2); i += 256) b4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        for (int64_t t = t0 + threadIdx.x; t < t1; t += 256) {
            const int64_t i = src[t] - a;
            if (i >= 0 && i < len) buf[i] = dy[t];
        }
        __syncthreads();
        // stream [a, b) out: scalar head up to 16-byte alignment, float4 body, scalar tail
        const int64_t head = min(len, (int64_t)((4 - (a & 3)) & 3));
        if (threadIdx.x < head) dx[a + threadIdx.x] = buf[threadIdx.x];
        const int64_t nb4 = (len - head) >> 2;
        for (int64_t q = threadIdx.x; q < nb4; q += 256) {
            const int64_t o = head + 4 * q;
            *reinterpret_cast<float4*>(dx + a + o) = make_float4(buf[o], buf[o + 1], buf[o + 2], buf[o + 3]);
        }
        for (int64_t r = head + 4 * nb4 + threadIdx.x; r < len; r += 256) dx[a + r] = buf[r];
        return;
    }
    const int lane = threadIdx.x & 31;
    // warp-uniform trip count (the long-gap path needs every lane); t = n is the tail sentinel
    const int64_t tend = last ? n + 1 : t1;
    for (int64_t w0 = t0 + (threadIdx.x & ~31); w0 < tend; w0 += 256) {
        const int64_t t = w0 + lane;
        int64_t lo = 0, hi = 0;   // zero [lo, hi)
        float v = 0.0f;
        if (t < tend) {
            lo = t == 0 ? 0 : clampi(src[t - 1] + 1);
            hi = t < n ? clampi(src[t]) : n_in;
            if (hi < lo) hi = lo;
            if (t < n) v = dy[t];
        }
        const bool longgap = hi - lo >= 64;
        if (!longgap)
            for (int64_t i = lo; i < hi; ++i) dx[i] = 0.0f;
        unsigned m = __ballot_sync(kFull, longgap);
        while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1;
            const int64_t l = __shfl_sync(kFull, lo, j), h = __shfl_sync(kFull, hi, j);
            const int64_t al = (l + 3) & ~(int64_t)3, ah = h & ~(int64_t)3;
            for (int64_t i = l + lane; i < al; i += 32) dx[i] = 0.0f;
            for (int64_t q = al + 4 * lane; q < ah; q += 128) *reinterpret_cast<float4*>(dx + q) = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int64_t i = ah + lane; i < h; i += 32) dx[i] = 0.0f;
        }
        if (t < n && src[t] >= 0 && src[t] < n_in) dx[src[t]] = v;
    }
}

__global__ void check_sorted_kernel(const int64_t* __restrict__ src, int64_t nbound, const int64_t* n_dev,
                                    int64_t n_in, int* flag) {
    const int64_t n = load_n(n_dev, nbound);
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = src[t];
        if (i < 0 || i >= n_in || (t > 0 && src[t - 1] >= i)) atomicOr(flag, 1);
    }
}

cudaError_t launch_check_sorted(const int64_t* src, int64_t n_out_bound, const int64_t* n_out_dev, int64_t n_in,
                                int* flag, cudaStream_t s) {
    if (n_out_bound <= 0) return cudaSuccess;
    const int64_t grid = std::min<int64_t>((n_out_bound + 255) / 256, num_sms() * 8);
    { SPC_PHASE("validate", s, 1); check_sorted_kernel<<<(unsigned)grid, 256, 0, s>>>(src, n_out_bound, n_out_dev, n_in, flag); }
    return cudaGetLastError();
}

cudaError_t launch_scatter_grad_sorted(const int64_t* src, const float* dy, int64_t n_out_bound,
                                       const int64_t* n_out_dev, float* dx, int64_t n_in, cudaStream_t s) {
    // one CTA per T sources plus the tail sentinel; T as large as keeps >= 4 CTAs per SM busy
    const int64_t want = 4 * (int64_t)num_sms();
    int items = 8;
    while (items > 1 && (n_out_bound + 1) / (256 * items) < want) items >>= 1;
    const unsigned grid = (unsigned)((n_out_bound + 256 * items) / (256 * items));
    SPC_PHASE("scatter_grad", s, 1);
    switch (items) {
        case 8: scatter_grad_sorted_kernel<2048><<<grid, 256, 0, s>>>(src, dy, n_out_bound, n_out_dev, dx, n_in); break;
        case 4: scatter_grad_sorted_kernel<1024><<<grid, 256, 0, s>>>(src, dy, n_out_bound, n_out_dev, dx, n_in); break;
        case 2: scatter_grad_sorted_kernel<512><<<grid, 256, 0, s>>>(src, dy, n_out_bound, n_out_dev, dx, n_in); break;
        default: scatter_grad_sorted_kernel<256><<<grid, 256, 0, s>>>(src, dy, n_out_bound, n_out_dev, dx, n_in); break;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------- sparseToDense bridge
// Table 2 "sparseToDense()": the key layout ((b*C + c)*V + row_major(p)) (reading R11)
// is the linear index of the dense [B, C, dims] tensor, so the bridge is a zero fill plus a
// scatter of the stored values; its backward gathers the dense gradient at the stored keys.
__global__ void to_dense_kernel(Keys keys, const float* __restrict__ vals,
                                const int64_t* nnz_dev, int64_t bound, float* __restrict__ dense) {
    const int64_t n = load_n(nnz_dev, bound);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dense[keys[i]] = vals[i];
}

__global__ void gather_dense_kernel(Keys keys, const int64_t* nnz_dev, int64_t bound,
                                    const float* __restrict__ ddense, float* __restrict__ dvals) {
    const int64_t n = load_n(nnz_dev, bound);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dvals[i] = ddense[keys[i]];
}

cudaError_t launch_to_dense(Keys keys, const float* vals, const int64_t* nnz_dev, int64_t bound,
                            float* dense, int64_t cells, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(dense, 0, (size_t)cells * sizeof(float), s);
    if (e != cudaSuccess || bound == 0) return e;
    const unsigned grid = (unsigned)std::min<int64_t>((bound + 255) / 256, num_sms() * 16);
    { SPC_PHASE("to_dense", s, 1); to_dense_kernel<<<grid, 256, 0, s>>>(keys, vals, nnz_dev, bound, dense); }
    return cudaGetLastError();
}

cudaError_t launch_gather_dense(Keys keys, const int64_t* nnz_dev, int64_t bound, const float* ddense,
                                float* dvals, cudaStream_t s) {
    if (bound == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<int64_t>((bound + 255) / 256, num_sms() * 16);
    { SPC_PHASE("gather_dense", s, 1); gather_dense_kernel<<<grid, 256, 0, s>>>(keys, nnz_dev, bound, ddense, dvals); }
    return cudaGetLastError();
}

// 32-bit key storage (Table 1 "Sparse 32"): the low word of every key; valid
// because the caller checked batch*channels*V < 2^32. Elementwise HBM streams.
__global__ void keys_narrow_kernel(const uint64_t* __restrict__ k, const int64_t* nnz_dev, int64_t bound,
                                   uint32_t* __restrict__ o) {
    const int64_t n = load_n(nnz_dev, bound);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        o[i] = (uint32_t)__ldcs(&k[i]);
}
__global__ void keys_widen_kernel(const uint32_t* __restrict__ k, const int64_t* nnz_dev, int64_t bound,
                                  uint64_t* __restrict__ o) {
    const int64_t n = load_n(nnz_dev, bound);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        o[i] = (uint64_t)__ldcs(&k[i]);
}

// Key codec (reading R11): one thread per entry; the decode divides by the extents
// from the last (least significant) dimension up, in 32-bit arithmetic when the key space fits.
__global__ void encode_keys_kernel(CodecGeo g, const int64_t* __restrict__ coords, int64_t n,
                                   uint64_t* __restrict__ keys, int* __restrict__ bad) {
    const int w = 2 + g.nd;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t* c = coords + i * w;
        const int64_t b = c[0], ch = c[1];
        bool ok = b >= 0 && b < g.B && ch >= 0 && ch < g.C;
        uint64_t lin = 0;
        for (int d = 0; d < g.nd; ++d) {
            const int64_t p = c[2 + d];
            ok = ok && p >= 0 && p < g.d[d];
            lin = lin * (uint64_t)g.d[d] + (uint64_t)(p >= 0 ? p : 0);
        }
        if (ok) {
            keys[i] = ((uint64_t)b * (uint64_t)g.C + (uint64_t)ch) * g.V + lin;
        } else {
            keys[i] = ~0ull;
            if (bad) *bad = 1;
        }
    }
}

template <typename U>
__global__ void decode_keys_kernel(CodecGeo g, const uint64_t* __restrict__ keys, int64_t n,
                                   int64_t* __restrict__ coords, int* __restrict__ bad) {
    const int w = 2 + g.nd;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[i];
        int64_t* c = coords + i * w;
        if (key >= g.total) {
            for (int d = 0; d < w; ++d) c[d] = -1;
            if (bad) *bad = 1;
            continue;
        }
        U r = (U)key;
        for (int d = g.nd - 1; d >= 0; --d) {
            const U q = r / (U)g.d[d];
            c[2 + d] = (int64_t)(r - q * (U)g.d[d]);
            r = q;
        }
        const U bb = r / (U)g.C;
        c[1] = (int64_t)(r - bb * (U)g.C);
        c[0] = (int64_t)bb;
    }
}

cudaError_t launch_encode_keys(const CodecGeo& g, const int64_t* coords, int64_t n, uint64_t* keys, int* bad,
                               cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, num_sms() * 16);
    { SPC_PHASE("encode_keys", s, 1); encode_keys_kernel<<<grid, 256, 0, s>>>(g, coords, n, keys, bad); }
    return cudaGetLastError();
}
cudaError_t launch_decode_keys(const CodecGeo& g, const uint64_t* keys, int64_t n, int64_t* coords, int* bad,
                               cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, num_sms() * 16);
    SPC_PHASE("decode_keys", s, 1);
    if (g.total <= 0xffffffffull) decode_keys_kernel<uint32_t><<<grid, 256, 0, s>>>(g, keys, n, coords, bad);
    else decode_keys_kernel<uint64_t><<<grid, 256, 0, s>>>(g, keys, n, coords, bad);
    return cudaGetLastError();
}

cudaError_t launch_keys_narrow(const uint64_t* keys, const int64_t* nnz_dev, int64_t bound, uint32_t* out, cudaStream_t s) {
    if (bound == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<int64_t>((bound + 255) / 256, num_sms() * 16);
    { SPC_PHASE("keys_narrow", s, 1); keys_narrow_kernel<<<grid, 256, 0, s>>>(keys, nnz_dev, bound, out); }
    return cudaGetLastError();
}
cudaError_t launch_keys_widen(const uint32_t* keys, const int64_t* nnz_dev, int64_t bound, uint64_t* out, cudaStream_t s) {
    if (bound == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<int64_t>((bound + 255) / 256, num_sms() * 16);
    { SPC_PHASE("keys_widen", s, 1); keys_widen_kernel<<<grid, 256, 0, s>>>(keys, nnz_dev, bound, out); }
    return cudaGetLastError();
}

}  // namespace spc

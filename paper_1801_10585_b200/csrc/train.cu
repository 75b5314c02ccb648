// Training-loop steps over the sparse filter bank: the adaptive density
// regulariser of §3.5 / Eq. (6) folded into an Adagrad step (§4), and one-warning-shot pruning
// (§3.6) as an order-preserving compaction of the filter COO. Both are elementwise over the
// stored weights, so pruned weights -- which are simply absent ("zero" = not stored) --
// never move and never come back.
#include "spc_internal.cuh"
#include "block_scan.cuh"

#include <algorithm>

namespace spc {

// Eq. (6), in double: b = o + b1 (rho - rho_up) above the bound, -b2 (rho_up - rho) below.
__device__ __forceinline__ double density_bias(double rho, const DensityReg& r) {
    return rho > r.rho_up ? __dadd_rn(r.o, __dmul_rn(r.b1, __dsub_rn(rho, r.rho_up)))
                          : -__dmul_rn(r.b2, __dsub_rn(r.rho_up, rho));
}

// One Adagrad step per stored parameter with the regulariser gradient 2*lambda*(w + b) added to
// the data gradient ("the regulariser becomes sum (w+b)^2"). The layer density rho is the
// forward output's count (device word) over its cell count, so no host synchronisation is needed.
// Double precision with explicit round-to-nearest operations (no contraction): the same sequence
// of IEEE operations as the oracle.
__global__ void adagrad_kernel(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ acc, int64_t n,
                               const int64_t* __restrict__ y_nnz_dev, double y_cells, DensityReg reg, int has_reg,
                               double lr, double eps) {
    double b = 0.0, lam = 0.0;
    if (has_reg) {
        const double rho = __ddiv_rn((double)*y_nnz_dev, y_cells);
        b = density_bias(rho, reg);
        lam = reg.lambda;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double wi = (double)w[i];
        const double gi = __dadd_rn((double)g[i], __dmul_rn(__dmul_rn(2.0, lam), __dadd_rn(wi, b)));
        const double a = __dadd_rn((double)acc[i], __dmul_rn(gi, gi));
        const double wn = __dsub_rn(wi, __ddiv_rn(__dmul_rn(lr, gi), __dadd_rn(__dsqrt_rn(a), eps)));
        acc[i] = (float)a;
        w[i] = (float)wn;
    }
}

cudaError_t launch_adagrad(float* w, const float* g, float* acc, int64_t n, const int64_t* y_nnz_dev, double y_cells,
                           const DensityReg& reg, bool has_reg, double lr, double eps, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, num_sms() * 8);
    { SPC_PHASE("adagrad", s, 1); adagrad_kernel<<<grid, 256, 0, s>>>(w, g, acc, n, y_nnz_dev, y_cells, reg, has_reg ? 1 : 0, lr, eps); }
    return cudaGetLastError();
}

// One-warning-shot pruning (§3.6): |w| < eps with the warning flag set -> removed;
// |w| < eps otherwise -> flag set; |w| >= eps -> flag cleared. Keys, values, accumulators and
// flags are compacted together in key order (count / device scan / write).
constexpr int kPrThreads = 256;
constexpr int kPrItems = 8;
constexpr int kPrChunk = kPrThreads * kPrItems;

__device__ __forceinline__ bool pr_keep(float w, uint8_t warn, double eps) {
    return !(fabs((double)w) < eps && warn);
}

__global__ void __launch_bounds__(kPrThreads) prune_count_kernel(const float* __restrict__ w, const uint8_t* __restrict__ warn,
                                                                  int64_t n, double eps, uint32_t* __restrict__ cnt) {
    const int64_t base = (int64_t)blockIdx.x * kPrChunk;
    uint32_t c = 0;
#pragma unroll
    for (int u = 0; u < kPrItems; ++u) {
        const int64_t i = base + (int64_t)u * kPrThreads + threadIdx.x;
        if (i < n) c += pr_keep(w[i], warn[i], eps);
    }
    __shared__ uint32_t sm[33];
    const uint32_t tot = block_sum(c, sm);
    if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kPrThreads) prune_write_kernel(const uint64_t* __restrict__ keys, const float* __restrict__ w,
                                                                  const float* __restrict__ acc, const uint8_t* __restrict__ warn,
                                                                  int64_t n, double eps, const uint64_t* __restrict__ off,
                                                                  uint64_t* __restrict__ ok, float* __restrict__ ow,
                                                                  float* __restrict__ oacc, uint8_t* __restrict__ owarn) {
    const int64_t base = (int64_t)blockIdx.x * kPrChunk;
    const int64_t my = base + (int64_t)threadIdx.x * kPrItems;
    uint32_t c = 0;
#pragma unroll
    for (int u = 0; u < kPrItems; ++u)
        if (my + u < n) c += pr_keep(w[my + u], warn[my + u], eps);
    __shared__ uint32_t sm[33];
    uint32_t tot;
    uint64_t pos = off[blockIdx.x] + block_excl_scan(c, sm, &tot);
#pragma unroll
    for (int u = 0; u < kPrItems; ++u) {
        const int64_t i = my + u;
        if (i < n && pr_keep(w[i], warn[i], eps)) {
            ok[pos] = keys[i];
            ow[pos] = w[i];
            if (oacc) oacc[pos] = acc[i];
            owarn[pos] = fabs((double)w[i]) < eps ? 1 : 0;
            ++pos;
        }
    }
}

size_t prune_ws_words(int64_t n) {
    const int64_t nch = (n + kPrChunk - 1) / kPrChunk;
    return (size_t)nch * 3 + scan_tmp_words(nch) + 8;
}

cudaError_t launch_prune(const uint64_t* keys, const float* w, const float* acc, const uint8_t* warn, int64_t n,
                         double eps, uint64_t* ok, float* ow, float* oacc, uint8_t* owarn, int64_t* out_nnz,
                         uint64_t* ws, cudaStream_t s) {
    const int64_t nch = (n + kPrChunk - 1) / kPrChunk;
    if (nch == 0) return cudaMemsetAsync(out_nnz, 0, sizeof(int64_t), s);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(ws);
    uint64_t* off = ws + nch;   // after nch u32 counts (<= nch u64 words)
    uint64_t* tmp = off + nch + 1;
    { SPC_PHASE("prune_count", s, 1); prune_count_kernel<<<(unsigned)nch, kPrThreads, 0, s>>>(w, warn, n, eps, cnt); }
    cudaError_t e = launch_scan_u32(cnt, off, nch, out_nnz, tmp, s);
    if (e != cudaSuccess) return e;
    { SPC_PHASE("prune_write", s, 1); prune_write_kernel<<<(unsigned)nch, kPrThreads, 0, s>>>(keys, w, acc, warn, n, eps, off, ok, ow, oacc, owarn); }
    return cudaGetLastError();
}

}  // namespace spc

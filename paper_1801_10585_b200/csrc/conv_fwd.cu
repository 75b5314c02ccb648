// Forward direct sparse convolution, Alg. 1 steps "for ic / for {id,val} / for
// {fid,fval}: atomically add val*fval to buffer at uid" and "add bias to non-zero entries".
//
// B200 mapping: the paper's temporary dense buffer per (b, oc) lives in
// global memory and receives global fp32 atomics one (b, oc) at a time.
// Here every (b, spatial tile, group of output channels) is a CTA whose slice of the buffer
// sits in shared memory; all (b, oc) run concurrently. A warp takes one input row (the Z
// entries of the last spatial dimension that share (b, ic, x, y)), its lanes take the stored
// weights of (oc-group, ic) and the warp walks the row's entries, so the 32 updates of one
// step hit 32 distinct (oc, voxel) targets. The buffer words start as an absent marker
// (kAbsent) and the CAS-based add replaces it on the first update: the structural support
// (reading R3) is recorded by the same atomic, without a second bitmap.
#include "spc_internal.cuh"
#include "block_scan.cuh"

namespace spc {

constexpr int kFwdThreads = 256;
constexpr size_t kFwdAccBudget = 96 * 1024;

ConvTile plan_fwd_tile(const Geo& gy, const KGeo& kg, int c_out) {
    ConvTile t{};
    int ocg = c_out < 16 ? c_out : 16;
    const size_t zb = (size_t)gy.Z * sizeof(float);
    while (ocg > 1 && zb * ocg * 4 > kFwdAccBudget) ocg = (ocg + 1) / 2;
    int64_t rows_max = (int64_t)(kFwdAccBudget / (zb * ocg));
    if (rows_max < 1) { t.smem = 0; return t; }   // row too long: unsupported
    const int64_t n_ocg = (c_out + ocg - 1) / ocg;
    // shrink tiles until there are enough CTAs to fill the machine twice
    for (;;) {
        double best = -1.0;
        int bx = 1, by = 1;
        for (int tx = 1; tx <= gy.X && tx <= rows_max; ++tx) {
            int ty = (int)(rows_max / tx);
            if (ty > gy.Y) ty = gy.Y;
            if (ty < 1) break;
            const double useful = (double)tx * ty;
            const double halo = (double)(tx + 2 * kg.hx) * (ty + 2 * kg.hy);
            const double score = useful / halo + 1e-6 * useful;
            if (score > best) { best = score; bx = tx; by = ty; }
        }
        t.TX = bx; t.TY = by;
        t.ntx = (gy.X + bx - 1) / bx;
        t.nty = (gy.Y + by - 1) / by;
        const int64_t ctas = (int64_t)t.ntx * t.nty * gy.B * n_ocg;
        if (ctas >= 2 * 148 || rows_max <= 1) break;
        rows_max /= 2;
    }
    t.ocg = ocg;
    t.n_ocg = (int)n_ocg;
    t.smem = (size_t)t.TX * t.TY * gy.Z * ocg * sizeof(float) + 64 * sizeof(unsigned);
    return t;
}

__device__ __forceinline__ void cas_add_absent(float* a, float v) {
    unsigned* p = reinterpret_cast<unsigned*>(a);
    unsigned old = *p, assumed;
    do {
        assumed = old;
        const float cur = (assumed == kAbsent) ? 0.0f : __uint_as_float(assumed);
        old = atomicCAS(p, assumed, __float_as_uint(cur + v));
    } while (old != assumed);
}

__global__ void __launch_bounds__(kFwdThreads)
conv_fwd_kernel(Geo gx, Geo gy, KGeo kg, ConvTile t, const uint64_t* __restrict__ xkeys,
                const float* __restrict__ xvals, const uint32_t* __restrict__ xrow,
                const int2* __restrict__ wmeta, const float* __restrict__ wval, const int* __restrict__ woff,
                const float* __restrict__ bias, float* __restrict__ pre, unsigned long long* __restrict__ seg_count) {
    extern __shared__ float acc[];                       // [ocg][TX*TY][Z]
    const int c_out = (int)gy.C;
    const int tix = blockIdx.x % t.ntx, tiy = blockIdx.x / t.ntx;
    const int64_t b = blockIdx.y;
    const int oc0 = blockIdx.z * t.ocg;
    const int nocl = min(t.ocg, c_out - oc0);
    const int x0 = tix * t.TX, y0 = tiy * t.TY;
    const int xe = min(x0 + t.TX, gy.X), ye = min(y0 + t.TY, gy.Y);
    const int Z = gy.Z;
    const int trows = t.TX * t.TY;
    const int ntile = trows * Z * t.ocg;
    unsigned* cnt = reinterpret_cast<unsigned*>(acc + ntile);
    for (int i = threadIdx.x; i < ntile; i += blockDim.x) reinterpret_cast<unsigned*>(acc)[i] = kAbsent;
    if (threadIdx.x < 64) cnt[threadIdx.x] = 0;
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int HX = t.TX + 2 * kg.hx, HY = t.TY + 2 * kg.hy;
    const int nh = HX * HY;
    const int c_in = (int)gx.C;
    for (int ic = 0; ic < c_in; ++ic) {
        const int wlo = woff[ic * (c_out + 1) + oc0];
        const int nwi = woff[ic * (c_out + 1) + oc0 + nocl] - wlo;
        if (nwi == 0) continue;
        for (int item = warp; item < nh; item += nwarps) {
            const int xs = x0 - kg.hx + item / HY;
            const int ys = y0 - kg.hy + item % HY;
            if (xs < 0 || xs >= gx.X || ys < 0 || ys >= gx.Y) continue;
            const int64_t row = ((b * c_in + ic) * gx.X + xs) * (int64_t)gx.Y + ys;
            const uint32_t e0 = xrow[row], e1 = xrow[row + 1];
            if (e0 == e1) continue;
            const uint64_t rowbase = (uint64_t)row * (uint64_t)Z;
            for (uint32_t eb = e0; eb < e1; eb += 32) {
                const int ne = (int)min(32u, e1 - eb);
                int zl = 0;
                float vl = 0.0f;
                if (lane < ne) {
                    zl = (int)(xkeys[eb + lane] - rowbase);
                    vl = xvals[eb + lane];
                }
                for (int wr = 0; wr < nwi; wr += 32) {
                    const int j = wr + lane;
                    bool ok = false;
                    int base = 0, oz = 0;
                    float w = 0.0f;
                    if (j < nwi) {
                        const int2 m = wmeta[wlo + j];
                        w = wval[wlo + j];
                        const int tx = xs - off_x(m.y), ty = ys - off_y(m.y);   // uid = id - (fid - centre)
                        oz = off_z(m.y);
                        ok = tx >= x0 && tx < xe && ty >= y0 && ty < ye;
                        base = ((m.x - oc0) * trows + (tx - x0) * t.TY + (ty - y0)) * Z;
                    }
                    if (!__any_sync(kFull, ok)) continue;
                    for (int e = 0; e < ne; ++e) {
                        const int z = __shfl_sync(kFull, zl, e);
                        const float v = __shfl_sync(kFull, vl, e);
                        const int tz = z - oz;
                        if (ok && tz >= 0 && tz < Z) cas_add_absent(&acc[base + tz], v * w);
                    }
                }
            }
        }
    }
    __syncthreads();
    // epilogue: bias on the support (Alg. 1 "add bias to non-zero entries"), write the
    // pre-attention slice to the (b, oc) buffers, count the support per (b, oc).
    for (int i = threadIdx.x; i < ntile; i += blockDim.x) {
        const int ocl = i / (trows * Z);
        const int rem = i - ocl * trows * Z;
        const int lr = rem / Z, z = rem - (rem / Z) * Z;
        const int x = x0 + lr / t.TY, y = y0 + lr % t.TY;
        if (ocl >= nocl || x >= gy.X || y >= gy.Y) continue;
        const int oc = oc0 + ocl;
        const unsigned bits = reinterpret_cast<unsigned*>(acc)[i];
        float out = __uint_as_float(kAbsent);
        if (bits != kAbsent) {
            out = __uint_as_float(bits) + (bias ? bias[oc] : 0.0f);
            atomicAdd(&cnt[ocl], 1u);
        }
        pre[(((b * c_out + oc) * gy.X + x) * (int64_t)gy.Y + y) * Z + z] = out;
    }
    __syncthreads();
    if (threadIdx.x < nocl && cnt[threadIdx.x])
        atomicAdd(&seg_count[b * c_out + oc0 + threadIdx.x], (unsigned long long)cnt[threadIdx.x]);
}

cudaError_t launch_conv_fwd(const Geo& gx, const Geo& gy, const KGeo& kg, const ConvTile& t,
                            const uint64_t* xkeys, const float* xvals, const uint32_t* xrow,
                            const int2* wmeta, const float* wval, const int* woff, const float* bias,
                            float* pre, unsigned long long* seg_count, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(conv_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t.smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)(t.ntx * t.nty), (unsigned)gy.B, (unsigned)t.n_ocg);
    if (grid.x == 0 || grid.y == 0) return cudaSuccess;
    { SPC_PHASE("conv_fwd", s, 1); conv_fwd_kernel<<<grid, kFwdThreads, t.smem, s>>>(gx, gy, kg, t, xkeys, xvals, xrow, wmeta, wval, woff, bias,
                                                      pre, seg_count); }
    return cudaGetLastError();
}

}  // namespace spc

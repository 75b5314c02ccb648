// Backward of the sparse convolution, Alg. 2 with the masked rule of Eqs. (3)/(4)
// (P:121-129): gradients only at stored inputs (dx) and stored weights (dw).
//
// B200 mapping: Alg. 2 initialises a dense buffer with the gradients of
// (b, oc) and, for every (input, weight) pair, reads g at uid and atomically adds
// g*fval to bp_data and g*val to bp_filter. Here a persistent CTA owns a group of
// output channels and walks (b, spatial tile) work items: the gradients of the tile plus its
// halo are scattered into a dense shared-memory buffer (zeros elsewhere = attention-dropped or
// non-existent outputs, reading R10), each lane owns one stored input entry and accumulates
// its dx in a register over all stored weights (no atomics on bp_data), and the dw
// contributions go to a per-CTA fp64 shared array that is flushed once per CTA. Lanes visit
// the weights in a lane-rotated order so that the 32 shared-memory updates of one step hit 32
// different weights.
#include "spc_internal.cuh"
#include "block_scan.cuh"

#include <algorithm>

namespace spc {

constexpr int kBwdThreads = 256;
constexpr size_t kBwdBudget = 200 * 1024;

BwdTile plan_bwd_tile(const Geo& gx, const KGeo& kg, int c_out, int nw_total) {
    BwdTile t{};
    const int c_in = (int)gx.C;
    const int zr = gx.Z + 2 * kg.hz;
    int ocg = c_out < 16 ? c_out : 16;
    for (;;) {
        const int64_t nwg = std::min<int64_t>((int64_t)nw_total, (int64_t)ocg * c_in * kg.KV);
        const size_t dwb = (size_t)nwg * sizeof(double) + (size_t)(c_in + 1) * sizeof(int) + 64;
        const size_t rowb = (size_t)zr * ocg * sizeof(float);
        if (dwb + rowb * (1 + 2 * kg.hx) * (1 + 2 * kg.hy) <= kBwdBudget || ocg == 1) {
            const int64_t hrows = dwb >= kBwdBudget ? 0 : (int64_t)((kBwdBudget - dwb) / rowb);
            double best = -1.0;
            int bx = 1, by = 1;
            for (int tx = 1; tx <= gx.X; ++tx) {
                if ((int64_t)(tx + 2 * kg.hx) * (1 + 2 * kg.hy) > hrows) break;
                int ty = (int)(hrows / (tx + 2 * kg.hx)) - 2 * kg.hy;
                if (ty > gx.Y) ty = gx.Y;
                if (ty < 1) break;
                const double score = (double)tx * ty / ((double)(tx + 2 * kg.hx) * (ty + 2 * kg.hy)) + 1e-6 * tx * ty;
                if (score > best) { best = score; bx = tx; by = ty; }
            }
            if (best < 0) { t.smem = 0; return t; }   // does not fit: unsupported
            t.TX = bx;
            t.TY = by;
            t.ocg = ocg;
            t.n_ocg = (c_out + ocg - 1) / ocg;
            t.ntx = (gx.X + bx - 1) / bx;
            t.nty = (gx.Y + by - 1) / by;
            const size_t gb = (size_t)(bx + 2 * kg.hx) * (by + 2 * kg.hy) * rowb;
            t.smem = gb + dwb;
            const int per_sm = (int)std::max<size_t>(1, (228 * 1024) / (t.smem + 1024));
            const int64_t items = gx.B * t.ntx * t.nty;
            int64_t grid = (int64_t)148 * std::min(per_sm, 8) / t.n_ocg;
            if (grid < 1) grid = 1;
            if (grid > items) grid = items;
            t.grid = (int)grid;
            return t;
        }
        ocg = (ocg + 1) / 2;
    }
}

__global__ void __launch_bounds__(kBwdThreads)
conv_bwd_kernel(Geo gx, Geo gy, KGeo kg, BwdTile t, const uint64_t* __restrict__ xkeys,
                const float* __restrict__ xvals, const uint32_t* __restrict__ xrow,
                const uint64_t* __restrict__ ykeys, const float* __restrict__ dy, const uint32_t* __restrict__ yrow,
                const int2* __restrict__ wmeta, const float* __restrict__ wval, const int* __restrict__ woff,
                const int* __restrict__ wsrc, float* __restrict__ dx, double* __restrict__ dw_acc,
                int want_dx, int want_dw) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int c_in = (int)gx.C, c_out = (int)gy.C;
    const int oc0 = blockIdx.y * t.ocg;
    const int nocl = min(t.ocg, c_out - oc0);
    const int HX = t.TX + 2 * kg.hx, HY = t.TY + 2 * kg.hy;
    const int ZR = gx.Z + 2 * kg.hz;
    const int hrows = HX * HY;
    const int gsize = t.ocg * hrows * ZR;
    // layout: dwp (double) | lbase (int c_in+1) | G (float)
    double* dwp = reinterpret_cast<double*>(smraw);
    // local weight bases per ic for this oc group (every thread computes nwg: c_in reads)
    int nwg = 0;
    for (int ic = 0; ic < c_in; ++ic)
        nwg += woff[ic * (c_out + 1) + oc0 + nocl] - woff[ic * (c_out + 1) + oc0];
    int* lbase = reinterpret_cast<int*>(smraw + (size_t)nwg * sizeof(double));
    float* G = reinterpret_cast<float*>(smraw + (((size_t)nwg * sizeof(double) + (size_t)(c_in + 1) * sizeof(int) + 15) & ~(size_t)15));
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int ic = 0; ic < c_in; ++ic) {
            lbase[ic] = acc;
            acc += woff[ic * (c_out + 1) + oc0 + nocl] - woff[ic * (c_out + 1) + oc0];
        }
        lbase[c_in] = acc;
    }
    for (int i = threadIdx.x; i < nwg; i += blockDim.x) dwp[i] = 0.0;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int64_t items = gx.B * (int64_t)t.ntx * t.nty;
    for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
        const int64_t b = item / ((int64_t)t.ntx * t.nty);
        const int tile = (int)(item - b * (int64_t)t.ntx * t.nty);
        const int x0 = (tile % t.ntx) * t.TX, y0 = (tile / t.ntx) * t.TY;
        __syncthreads();
        for (int i = threadIdx.x; i < gsize; i += blockDim.x) G[i] = 0.0f;
        __syncthreads();
        // "initialize dense buffer with gradients(b, oc)", restricted to tile + halo
        for (int r = warp; r < nocl * hrows; r += nwarps) {
            const int ocl = r / hrows, hr = r - ocl * hrows;
            const int xs = x0 - kg.hx + hr / HY, ys = y0 - kg.hy + hr % HY;
            if (xs < 0 || xs >= gy.X || ys < 0 || ys >= gy.Y) continue;
            const int64_t row = ((b * c_out + oc0 + ocl) * gy.X + xs) * (int64_t)gy.Y + ys;
            const uint32_t e0 = yrow[row], e1 = yrow[row + 1];
            const uint64_t rowbase = (uint64_t)row * (uint64_t)gy.Z;
            for (uint32_t e = e0 + lane; e < e1; e += 32)
                G[(ocl * hrows + hr) * ZR + (int)(ykeys[e] - rowbase) + kg.hz] = dy[e];
        }
        __syncthreads();
        const int xe = min(x0 + t.TX, gx.X), ye = min(y0 + t.TY, gx.Y);
        const int nrow = (xe - x0) * (ye - y0);
        for (int ic = 0; ic < c_in; ++ic) {
            const int wlo = woff[ic * (c_out + 1) + oc0];
            const int nwi = woff[ic * (c_out + 1) + oc0 + nocl] - wlo;
            if (nwi == 0) continue;
            const int lb = lbase[ic];
            for (int rr = warp; rr < nrow; rr += nwarps) {
                const int x = x0 + rr / (ye - y0), y = y0 + rr % (ye - y0);
                const int64_t row = ((b * c_in + ic) * gx.X + x) * (int64_t)gx.Y + y;
                const uint32_t e0 = xrow[row], e1 = xrow[row + 1];
                const uint64_t rowbase = (uint64_t)row * (uint64_t)gx.Z;
                const int hxr = x - x0 + kg.hx, hyr = y - y0 + kg.hy;
                for (uint32_t e = e0 + lane; e < e1; e += 32) {
                    const int z = (int)(xkeys[e] - rowbase);
                    const float v = xvals[e];
                    float dxa = 0.0f;
                    int j = lane % nwi;
                    for (int jj = 0; jj < nwi; ++jj) {
                        const int2 m = wmeta[wlo + j];
                        // g at uid = id - (fid - centre)
                        const int gi = ((m.x - oc0) * hrows + (hxr - off_x(m.y)) * HY + (hyr - off_y(m.y))) * ZR +
                                       z - off_z(m.y) + kg.hz;
                        const float g = G[gi];
                        if (g != 0.0f) {
                            const float w = wval[wlo + j];
                            dxa = fmaf(g, w, dxa);                                   // bp_data += g*fval
                            if (want_dw) atomicAdd(&dwp[lb + j], (double)g * (double)v);  // bp_filter += g*val
                        }
                        j = (j + 1 == nwi) ? 0 : j + 1;
                    }
                    if (want_dx) {
                        if (t.n_ocg == 1) dx[e] = dxa;
                        else atomicAdd(&dx[e], dxa);
                    }
                }
            }
        }
    }
    __syncthreads();
    if (want_dw) {
        for (int ic = 0; ic < c_in; ++ic) {
            const int wlo = woff[ic * (c_out + 1) + oc0];
            const int n = lbase[ic + 1] - lbase[ic];
            for (int j = threadIdx.x; j < n; j += blockDim.x) {
                const double v = dwp[lbase[ic] + j];
                if (v != 0.0) atomicAdd(&dw_acc[wsrc[wlo + j]], v);
            }
        }
    }
}

cudaError_t launch_conv_bwd(const Geo& gx, const Geo& gy, const KGeo& kg, const BwdTile& t,
                            const uint64_t* xkeys, const float* xvals, const uint32_t* xrow,
                            const uint64_t* ykeys, const float* dy, const uint32_t* yrow,
                            const int2* wmeta, const float* wval, const int* woff, const int* wsrc,
                            float* dx, double* dw_acc, bool want_dx, bool want_dw, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(conv_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t.smem);
    if (e != cudaSuccess) return e;
    if (gx.B == 0) return cudaSuccess;
    dim3 grid((unsigned)t.grid, (unsigned)t.n_ocg);
    { SPC_PHASE("conv_bwd", s, 1); conv_bwd_kernel<<<grid, kBwdThreads, t.smem, s>>>(gx, gy, kg, t, xkeys, xvals, xrow, ykeys, dy, yrow, wmeta,
                                                      wval, woff, wsrc, dx, dw_acc, want_dx ? 1 : 0,
                                                      want_dw ? 1 : 0); }
    return cudaGetLastError();
}

// dbias[oc] = sum of dy over the kept outputs of oc (fp64 accumulation).
__global__ void dbias_kernel(Geo gy, const uint64_t* __restrict__ ykeys, const float* __restrict__ dy,
                             const int64_t* ny_dev, int64_t nbound, double* __restrict__ db) {
    extern __shared__ double sdb[];
    const int c_out = (int)gy.C;
    for (int i = threadIdx.x; i < c_out; i += blockDim.x) sdb[i] = 0.0;
    __syncthreads();
    const int64_t n = load_n(ny_dev, nbound);
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const int oc = (int)((ykeys[t] / (uint64_t)gy.V) % (uint64_t)c_out);
        atomicAdd(&sdb[oc], (double)dy[t]);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < c_out; i += blockDim.x)
        if (sdb[i] != 0.0) atomicAdd(&db[i], sdb[i]);
}

cudaError_t launch_dbias(const Geo& gy, const uint64_t* ykeys, const float* dy, const int64_t* ny_dev,
                         int64_t ny_bound, double* db_acc, cudaStream_t s) {
    if (ny_bound <= 0) return cudaSuccess;
    int64_t grid = (ny_bound + 255) / 256;
    if (grid > 592) grid = 592;
    const size_t sm = (size_t)gy.C * sizeof(double);
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(dbias_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
    }
    { SPC_PHASE("dbias", s, 1); dbias_kernel<<<(unsigned)grid, 256, sm, s>>>(gy, ykeys, dy, ny_dev, ny_bound, db_acc); }
    return cudaGetLastError();
}

}  // namespace spc

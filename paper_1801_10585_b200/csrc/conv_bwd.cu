// Backward of the sparse convolution, Alg. 2 with the masked rule of Eqs. (3)/(4)
// (P:121-129): gradients only at stored inputs (dx) and stored weights (dw).
//
// B200 mapping: Alg. 2 initialises a dense buffer with the
// gradients of (b, oc) and for every (input, weight) pair reads g at uid and atomically
// adds g*fval to bp_data and g*val to bp_filter. Here a persistent CTA owns a group
// of output channels and walks (b, spatial tile) items. The gradients of the tile plus halo are
// scattered into a zero shared-memory buffer G with margins (attention-dropped and absent
// outputs read 0, reading R10; out-of-grid targets land in the margin). The stored entries of
// the tile are processed in warp-level 32x32 blocks: lane L owns weight j0+L, the warp walks 32
// staged entries; g = G[ebase(e) - wdel(j)] is one shared load; lane L accumulates g*x into its
// dw register and the 32x32 products g*w are reduced across lanes with a shuffle
// reduce-scatter that leaves dx(e) in lane e. No atomics on dx inside a group; dw goes to a
// per-CTA fp64 shared array once per block and to global fp64 once per CTA.
#include "spc_internal.cuh"
#include "block_scan.cuh"

#include <algorithm>
#include <cstdlib>

namespace spc {

// CTA shapes: one 512-thread CTA per SM (largest G slab), or two 256-thread CTAs per SM that
// hide each other's per-item global-memory latency (SPC_BWD_CTAS=1|2 overrides the default)
static int bwd_ctas_per_sm() {
    const char* v = getenv("SPC_BWD_CTAS");
    return (v && v[0] == '2') ? 2 : 1;
}

// Strides of the G slab (floats): y-row sY, x-row sX, w-plane sW, output-channel slice sOC, each
// padded to a residue mod 32 that makes the filter offsets dz + dy*sY + dx*sX + dw*sW land in
// distinct banks (mixed radix kz, kz*ky, kz*ky*kx, ...): the 32 lanes of a G load read one
// entry's targets under 32 different weights, i.e. 32 different filter offsets.
struct BwdStrides {
    int sY, sX, sW, sOC;
};
static BwdStrides bwd_strides(const KGeo& kg, int Z, int TX, int TY) {
    auto pad = [](int v, int r) { return v + ((r - v) % 32 + 32) % 32; };   // >= v, == r mod 32
    const int HW = 1 + 2 * kg.hw, HX = TX + 2 * kg.hx, HY = TY + 2 * kg.hy;
    BwdStrides st;
    st.sY = pad(Z + 2 * kg.hz, kg.kz % 32);
    st.sX = pad(HY * st.sY, (kg.kz * kg.ky) % 32);
    st.sW = pad(HX * st.sX, (kg.kz * kg.ky * kg.kx) % 32);
    st.sOC = pad(HW * st.sW, (kg.kz * kg.ky * kg.kx * kg.kw) % 32);
    return st;
}

// ocs: output channels in the G slab (one pass); ocp passes per item cover the CTA's group
static size_t bwd_smem(const KGeo& kg, int c_in, int TX, int TY, int Z, int ocs, int ocp, int64_t nwg, int threads) {
    const size_t g = (size_t)ocs * bwd_strides(kg, Z, TX, TY).sOC * sizeof(float);
    const size_t w = (size_t)nwg * (sizeof(int) + sizeof(float) + sizeof(double));
    // lbase / cpre, and two buffers each of the entry-range bounds (rng) and the halo-row bounds
    // of the gradient fill (prefetched one item ahead)
    const size_t nhalo = (size_t)ocs * ocp * (1 + 2 * kg.hw) * (TX + 2 * kg.hx);
    const size_t idx = (size_t)(c_in + 1) * sizeof(int) * (1 + ocp) + 2 * (size_t)c_in * TX * 2 * sizeof(uint32_t) +
                       2 * nhalo * 2 * sizeof(uint32_t);
    const size_t stage = (size_t)(threads / 32) * 32 * 4 * sizeof(int);   // per warp: 4 x 32 words
    return g + w + idx + stage + 256;
}

static BwdTile plan_bwd_tile_ocp(const Geo& gx, const KGeo& kg, int c_out, int nw_total, int ocp_req) {
    BwdTile t{};
    const int c_in = (int)gx.C;
    const int cps = bwd_ctas_per_sm();
    const int threads = cps == 2 ? 256 : 512;
    const size_t budget = cps == 2 ? 110 * 1024 : 200 * 1024;
    int ocg = std::min(c_out, cps == 2 ? 4 : 8);
    for (; ocg >= 1; ocg = ocg > 1 ? (ocg + 1) / 2 : 0) {
        int ocp = std::min(ocp_req, ocg);
        while (ocg % ocp) --ocp;
        const int ocs = ocg / ocp;
        const int64_t nwg = std::min<int64_t>(nw_total, (int64_t)ocg * c_in * kg.KV);
        double best = -1.0;
        int bx = 0, by = 0;
        for (int tx = 1; tx <= gx.X && tx <= 64; ++tx) {
            int lo = 1, hi = gx.Y, ty = 0;
            while (lo <= hi) {   // largest ty that fits
                const int mid = (lo + hi) / 2;
                if (bwd_smem(kg, c_in, tx, mid, gx.Z, ocs, ocp, nwg, threads) <= budget) { ty = mid; lo = mid + 1; }
                else hi = mid - 1;
            }
            if (ty < 1) break;
            ty = std::min(ty, 64);
            const double score = (double)tx * ty / ((double)(tx + 2 * kg.hx) * (ty + 2 * kg.hy)) + 1e-9 * tx * ty;
            if (score > best) { best = score; bx = tx; by = ty; }
        }
        if (best < 0) { if (ocg == 1) break; continue; }
        t.TX = bx;
        t.TY = by;
        t.ocg = ocg;
        t.ocp = ocp;
        t.ocs = ocs;
        t.n_ocg = (c_out + ocg - 1) / ocg;
        t.ntx = (gx.X + bx - 1) / bx;
        t.nty = (gx.Y + by - 1) / by;
        t.nwg_max = (int)nwg;
        t.smem = bwd_smem(kg, c_in, bx, by, gx.Z, ocs, ocp, nwg, threads);
        {
            const BwdStrides st = bwd_strides(kg, gx.Z, bx, by);
            t.sY = st.sY;
            t.sX = st.sX;
            t.sW = st.sW;
            t.sOC = st.sOC;
        }
        t.threads = threads;
        const int64_t items = gx.B * gx.W * (int64_t)t.ntx * t.nty;
        int64_t grid = (num_sms() * cps + t.n_ocg - 1) / t.n_ocg;
        grid = std::max<int64_t>(1, std::min<int64_t>(grid, items));
        t.grid = (int)grid;
        if (items >= ((int64_t)1 << 31)) { t.smem = 0; return t; }   // 32-bit item decode
        const int HX = bx + 2 * kg.hx, HW = 1 + 2 * kg.hw;
        t.fd_tiles = make_fastdiv((uint32_t)(t.ntx * t.nty));
        t.fd_W = make_fastdiv((uint32_t)gx.W);
        t.fd_ntx = make_fastdiv((uint32_t)t.ntx);
        t.fd_HWX = make_fastdiv((uint32_t)(HW * HX));
        t.fd_HX = make_fastdiv((uint32_t)HX);
        t.fd_TX = make_fastdiv((uint32_t)bx);
        return t;
    }
    t.smem = 0;
    return t;
}

// Passes per item (SPC_BWD_OCP overrides): with ocp passes the G slab holds ocg / ocp channels,
// so the tile can be larger (less halo re-read per interior voxel, more entry chunks per item to
// spread over the warps) at the cost of ocp fills / sweeps per item. Two passes are taken for
// wide inputs (>= 32 channels) when they buy at least 1.5x the tile area. Measured: C4 (8 input
// channels) 3.12 / 3.69 ms with 1 / 2 passes; the C3 chain (32 -> 64 layer) 20.3 / 18.3 ms per
// step; C5 32 -> 32 at 50 % 20.1 -> 13.2 ms; C2 (16 -> 32 on 7 x 7 planes) 0.70 / 0.74 ms; the
// OctNet3 trunk (16 / 24 input channels) 8.66 / 9.15 ms.
BwdTile plan_bwd_tile(const Geo& gx, const KGeo& kg, int c_out, int nw_total) {
    if (const char* v = getenv("SPC_BWD_OCP")) return plan_bwd_tile_ocp(gx, kg, c_out, nw_total, std::max(1, atoi(v)));
    const BwdTile t1 = plan_bwd_tile_ocp(gx, kg, c_out, nw_total, 1);
    if (gx.C < 32 || t1.smem == 0) return t1;
    const BwdTile t2 = plan_bwd_tile_ocp(gx, kg, c_out, nw_total, 2);
    return (t2.smem && t2.ocp == 2 && (double)t2.TX * t2.TY >= 1.5 * t1.TX * t1.TY) ? t2 : t1;
}

// 32 values per lane -> lane L receives the sum over lanes of v[L] (butterfly reduce-scatter).
__device__ __forceinline__ float reduce_scatter32(float (&v)[32], int lane) {
#pragma unroll
    for (int half = 16; half >= 1; half >>= 1) {
        const bool up = (lane & half) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const float send = up ? v[i] : v[i + half];
            const float keep = up ? v[i + half] : v[i];
            v[i] = keep + __shfl_xor_sync(kFull, send, half);
        }
    }
    return v[0];
}

// Slot order of the weights of one (pass, input channel) range of the backward filter table: the
// lanes of conv_bwd_kernel walk a range in blocks of 32 weights, and two lanes of a block whose G
// offsets agree mod 32 words read the same shared-memory bank for every entry. So the range is
// reordered in place (before conv_bwd_kernel, once per call, one warp per range): weights sorted
// by the bank residue of their G offset (ties in table order), then position i of that order goes
// to block i % nb, lane i / nb while every block still has room (the last block holds
// L = n - 32 (nb - 1)), the rest round-robin over the full blocks. dw per weight is unaffected
// (each weight keeps its source index); dx(e), a sum over the weights, only changes its fp32
// summation order. Ranges of more than 256 weights keep the table order.
__global__ void __launch_bounds__(512) bwd_slot_order_kernel(KGeo kg, BwdTile t, int c_in, int c_out,
                                                             int2* __restrict__ wmeta, float* __restrict__ wval,
                                                             int* __restrict__ wsrc, const int* __restrict__ woff) {
    __shared__ int cnt_all[16][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int* cnt = cnt_all[warp];
    const int oc0 = blockIdx.x * t.ocg, nocl = min(t.ocg, c_out - oc0);
    const uint32_t lt = (1u << lane) - 1u;
    for (int q = warp; q < c_in * t.ocp; q += 16) {
        const int pp = q / c_in, ic = q - pp * c_in;
        const int ocb = oc0 + pp * t.ocs;
        const int t0 = woff[ic * (c_out + 1) + oc0 + min(nocl, pp * t.ocs)];
        const int n = woff[ic * (c_out + 1) + oc0 + min(nocl, (pp + 1) * t.ocs)] - t0;
        if (n <= 32 || n > 256) continue;   // one block (nothing to spread) / too long: table order
        const int nb = (n + 31) >> 5, L = n - 32 * (nb - 1);
        int2 mm[8];
        float vv[8];
        int ss[8], dd[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int j = c * 32 + lane;
            const bool ok = j < n;
            mm[c] = ok ? wmeta[t0 + j] : make_int2(0, 0);
            vv[c] = ok ? wval[t0 + j] : 0.0f;
            ss[c] = ok ? wsrc[t0 + j] : 0;
            // g at uid = id - (fid - centre): G index = ebase - wdel, as conv_bwd_kernel
            dd[c] = meta_ow(mm[c].x) * t.sW + off_x(mm[c].y) * t.sX + off_y(mm[c].y) * t.sY + off_z(mm[c].y) -
                    (meta_oc(mm[c].x) - ocb) * t.sOC;
        }
        cnt[lane] = 0;
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 8; ++c) {   // per-residue totals
            const bool ok = c * 32 + lane < n;
            const int r = ok ? (dd[c] & 31) : 32 + lane;
            const unsigned m = __match_any_sync(kFull, r);
            if (ok && (m >> lane) == 1u) cnt[r] += __popc(m);   // the highest lane of the residue group
            __syncwarp();
        }
        const int c0 = cnt[lane];
        const int incl = warp_incl_scan(c0);
        __syncwarp();
        cnt[lane] = incl - c0;   // first position of residue lane
        __syncwarp();
        int slot[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const bool ok = c * 32 + lane < n;
            const int r = ok ? (dd[c] & 31) : 32 + lane;
            const unsigned m = __match_any_sync(kFull, r);
            const int i = ok ? cnt[r] + __popc(m & lt) : 0;
            __syncwarp();
            if (ok && (m >> lane) == 1u) cnt[r] += __popc(m);
            __syncwarp();
            slot[c] = i < nb * L ? (i % nb) * 32 + i / nb
                                 : ((i - nb * L) % (nb - 1)) * 32 + L + (i - nb * L) / (nb - 1);
        }
        __syncwarp();   // every lane holds its weights: write them back in slot order
#pragma unroll
        for (int c = 0; c < 8; ++c)
            if (c * 32 + lane < n) {
                wmeta[t0 + slot[c]] = mm[c];
                wval[t0 + slot[c]] = vv[c];
                wsrc[t0 + slot[c]] = ss[c];
            }
    }
}

template <bool DX, bool DW, int THREADS>
__global__ void __launch_bounds__(THREADS, 512 / THREADS)
conv_bwd_kernel(Geo gx, Geo gy, KGeo kg, BwdTile t, Keys xkeys,
                const float* __restrict__ xvals, const uint32_t* __restrict__ xrow,
                Keys ykeys, const float* __restrict__ dy, const uint32_t* __restrict__ yrow,
                const int2* __restrict__ wmeta, const float* __restrict__ wval, const int* __restrict__ woff,
                const int* __restrict__ wsrc, float* __restrict__ dx, double* __restrict__ dw_acc) {
    extern __shared__ __align__(16) unsigned char smraw[];
    const int c_in = (int)gx.C, c_out = (int)gy.C;
    const int oc0 = blockIdx.y * t.ocg;
    const int nocl = min(t.ocg, c_out - oc0);
    // G slab of one output-channel slice: HW w-planes x HX x-rows x HY y-rows x ZR (rank-4 maps:
    // the tile is one w-plane, its halo the 2*hw neighbouring planes; HW = 1 for rank <= 3)
    // (strides t.sY / sX / sW / sOC: bwd_strides)
    const int HW = 1 + 2 * kg.hw, HX = t.TX + 2 * kg.hx;
    const int sY = t.sY, sX = t.sX, sW = t.sW, sOC = t.sOC;
    const int gsize = t.ocs * sOC;   // the slab holds the ocs channels of one pass
    const int ocp = t.ocp, ocs = t.ocs;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int nwarps = THREADS / 32;

    // ---- shared layout: G | dwp | wdel | wv | lbase | cpre | rng | stage
    float* G = reinterpret_cast<float*>(smraw);
    unsigned char* p = smraw + (((size_t)gsize * sizeof(float) + 15) & ~(size_t)15);
    double* dwp = reinterpret_cast<double*>(p);
    p += (size_t)t.nwg_max * sizeof(double);
    int* wdel = reinterpret_cast<int*>(p);
    p += (size_t)t.nwg_max * sizeof(int);
    float* wv = reinterpret_cast<float*>(p);
    p += (size_t)t.nwg_max * sizeof(float);
    int* lbase = reinterpret_cast<int*>(p);   // [pass][ic]: first slot of (pass, ic); [ocp*(c_in+1)]
    p += (size_t)(c_in + 1) * ocp * sizeof(int);
    int* cpre = reinterpret_cast<int*>(p);
    p += (size_t)(c_in + 1) * sizeof(int);
    uint32_t* rbuf[2];   // entry-range bounds per (ic, x-row) of an item, double-buffered
    rbuf[0] = reinterpret_cast<uint32_t*>(p);
    p += (size_t)c_in * t.TX * 2 * sizeof(uint32_t);
    rbuf[1] = reinterpret_cast<uint32_t*>(p);
    p += (size_t)c_in * t.TX * 2 * sizeof(uint32_t);
    const int nhalo = t.ocg * HW * HX;   // halo rows of the group (all passes)
    uint32_t* fbuf[2];   // per halo row the kept-output range of its y-rows, double-buffered
    fbuf[0] = reinterpret_cast<uint32_t*>(p);
    p += (size_t)nhalo * 2 * sizeof(uint32_t);
    fbuf[1] = reinterpret_cast<uint32_t*>(p);
    p += (size_t)nhalo * 2 * sizeof(uint32_t);
    // align from the __shared__ base with integer offsets (keeps the shared address space)
    p = smraw + ((size_t)(p - smraw + 15) & ~(size_t)15);
    int* st_eb = reinterpret_cast<int*>(p) + warp * 128;   // per warp: 32 ebase + 32 values (+ 64 fill words)
    float* st_v = reinterpret_cast<float*>(st_eb + 32);
    int* st_gb = st_eb + 64;                               // G fill: per halo row its G base ...
    uint32_t* st_rz = reinterpret_cast<uint32_t*>(st_eb + 96);   // ... and the low word of its first key

    // ---- one-time setup: group weights with their G-offsets, zero G and dw partials. The
    // weights of an input channel are walked by lanes in blocks of 32; two lanes of a block whose
    // G offsets agree mod 32 words read the same bank for every entry. So the weights of each
    // input channel are ordered by that residue and dealt round-robin to the channel's blocks
    // (bwd_slot): same-residue weights land in different blocks. dw per weight is unaffected by
    // the order; dx(e), a sum over the weights, only changes its fp32 summation order.
    // pass p covers output channels oc0 + p*ocs .. (its weights of input channel ic are the
    // contiguous range wo(p, ic) .. wo(p + 1, ic) of the filter table)
    auto wo = [&](int pp, int ic) { return woff[ic * (c_out + 1) + oc0 + min(nocl, pp * ocs)]; };
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int pp = 0; pp < ocp; ++pp) {
            for (int ic = 0; ic < c_in; ++ic) {
                lbase[pp * (c_in + 1) + ic] = acc;
                acc += wo(pp + 1, ic) - wo(pp, ic);
            }
            lbase[pp * (c_in + 1) + c_in] = acc;
        }
    }
    __syncthreads();
    const int nwg = lbase[(ocp - 1) * (c_in + 1) + c_in];
    for (int q = warp; q < c_in * ocp; q += nwarps) {   // one warp per (pass, input channel)
        const int pp = q / c_in, ic = q - pp * c_in;
        const int ocb = oc0 + pp * ocs;   // first channel of the pass: slice 0 of the slab
        const int lb = lbase[pp * (c_in + 1) + ic], t0 = wo(pp, ic), n = wo(pp + 1, ic) - t0;
        for (int j = lane; j < n; j += 32) {   // (the table range is in slot order: bwd_slot_order_kernel)
            const int2 m = wmeta[t0 + j];
            // g at uid = id - (fid - centre): G index = ebase - wdel
            wdel[lb + j] = meta_ow(m.x) * sW + off_x(m.y) * sX + off_y(m.y) * sY + off_z(m.y) - (meta_oc(m.x) - ocb) * sOC;
            wv[lb + j] = wval[t0 + j];
        }
    }
    for (int i = threadIdx.x; i < nwg; i += blockDim.x) dwp[i] = 0.0;
    for (int i = threadIdx.x; i < gsize; i += blockDim.x) G[i] = 0.0f;
    const int eb_safe = kg.hw * sW + kg.hx * sX + kg.hy * sY + kg.hz;   // an in-range G index for idle lanes

    const int64_t items = gx.B * gx.W * (int64_t)t.ntx * t.nty;
    const int HWX = HW * HX;
    const float invZ = 1.0f / (float)gy.Z;
    const float invXZ = 1.0f / (float)gx.Z;
    struct ItemGeo { int64_t b; int wp, x0, y0, xe, ye, hylo, hyhi; };
    auto item_geo = [&](int64_t item) {   // (items < 2^31, plan_bwd_tile): divisions by multiply-high
        ItemGeo g;
        const uint32_t bw = fdiv((uint32_t)item, t.fd_tiles);   // (b, w-plane)
        const uint32_t bq = fdiv(bw, t.fd_W);
        g.b = bq;
        g.wp = (int)(bw - bq * (uint32_t)gx.W);
        const int tile = (int)((uint32_t)item - bw * (uint32_t)(t.ntx * t.nty));
        const int tyi = (int)fdiv((uint32_t)tile, t.fd_ntx);
        g.x0 = (tile - tyi * t.ntx) * t.TX;
        g.y0 = tyi * t.TY;
        g.xe = min(g.x0 + t.TX, gx.X);
        g.ye = min(g.y0 + t.TY, gx.Y);
        g.hylo = max(0, g.y0 - kg.hy);
        g.hyhi = min(gy.Y, g.y0 + t.TY + kg.hy);
        return g;
    };
    // halo row r of the group = (ocl, hw-plane, hx-row) -> its first y-row in the output map (or
    // -1) and its base in the slab (channel slice ocl % ocs of its pass)
    auto halo_row = [&](const ItemGeo& g, int r, int& gbase) -> int64_t {
        const int ocl = (int)fdiv((uint32_t)r, t.fd_HWX), hr = r - ocl * HWX;
        const int hwi = (int)fdiv((uint32_t)hr, t.fd_HX), hxr = hr - hwi * HX;
        const int ws = g.wp - kg.hw + hwi, xs = g.x0 - kg.hx + hxr;
        gbase = (ocl % ocs) * sOC + hwi * sW + hxr * sX + (g.hylo - (g.y0 - kg.hy)) * sY + kg.hz;
        if (ws < 0 || ws >= gy.W || xs < 0 || xs >= gy.X || g.hylo >= g.hyhi || ocl >= nocl) return -1;
        return (((g.b * c_out + oc0 + ocl) * gy.W + ws) * gy.X + xs) * (int64_t)gy.Y + g.hylo;
    };
    // the bounds of an item, fetched with cp.async one item ahead (their latency overlaps the
    // current item): per (ic, x-row) the stored entries of rows y0..ye-1 (one contiguous run), per
    // halo row the kept outputs of its halo y-range (one contiguous run)
    auto cp4 = [](uint32_t* dst, const uint32_t* src) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;"
                     :: "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src) : "memory");
    };
    auto prefetch = [&](int64_t item, uint32_t* rb, uint32_t* fbb) {
        // (issued by the highest threads: warp 0 goes on with the chunk prefix meanwhile)
        const int tr = (int)blockDim.x - 1 - (int)threadIdx.x;
        const ItemGeo g = item_geo(item);
        for (int q = tr; q < c_in * t.TX; q += blockDim.x) {
            const int ic = (int)fdiv((uint32_t)q, t.fd_TX), xi = q - ic * t.TX;
            if (g.x0 + xi < g.xe) {
                const int64_t r0 = (((g.b * c_in + ic) * gx.W + g.wp) * gx.X + g.x0 + xi) * (int64_t)gx.Y + g.y0;
                cp4(rb + 2 * q, xrow + r0);
                cp4(rb + 2 * q + 1, xrow + r0 + (g.ye - g.y0));
            } else {
                rb[2 * q] = 0u;
                rb[2 * q + 1] = 0u;
            }
        }
        for (int r = tr; r < nhalo; r += blockDim.x) {
            int gb;
            const int64_t row = halo_row(g, r, gb);
            if (row >= 0) {
                cp4(fbb + 2 * r, yrow + row);
                cp4(fbb + 2 * r + 1, yrow + row + (g.hyhi - g.hylo));
            } else {
                fbb[2 * r] = 0u;
                fbb[2 * r + 1] = 0u;
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int cb = 0;
    if (blockIdx.x < items) prefetch(blockIdx.x, rbuf[0], fbuf[0]);
    for (int64_t item = blockIdx.x; item < items; item += gridDim.x, cb ^= 1) {
        const ItemGeo ig = item_geo(item);
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();   // this item's bounds are in; the previous item's sweep of G is complete
        if (item + gridDim.x < items) prefetch(item + gridDim.x, cb ? rbuf[0] : rbuf[1], cb ? fbuf[0] : fbuf[1]);
        const uint32_t* rng = cb ? rbuf[1] : rbuf[0];
        const uint32_t* fbd = cb ? fbuf[1] : fbuf[0];
        if (warp == 0) {   // chunks per ic (32 entries each), exclusive prefix over ic
            int carry = 0;
            for (int ic0 = 0; ic0 < c_in; ic0 += 32) {
                const int ic = ic0 + lane;
                int cnt = 0;
                if (ic < c_in)
                    for (int xi = 0; xi < t.TX; ++xi)
                        cnt += (int)(rng[2 * (ic * t.TX + xi) + 1] - rng[2 * (ic * t.TX + xi)]);
                const int nch = (cnt + 31) >> 5;
                const int incl = warp_incl_scan(nch);
                if (ic < c_in) cpre[ic] = carry + incl - nch;
                carry += __shfl_sync(kFull, incl, 31);
            }
            if (lane == 0) cpre[c_in] = carry;
        }
        __syncthreads();
        const int nchunks = cpre[c_in];
        // chunk f -> (ic, entry of this lane) from the shared ranges, and the entry's key and value
        // loads issued; the first chunk's loads are in flight during the gradient fill, the next
        // chunk's while this chunk's blocks run
        struct Loc { int ic, xi; int64_t e; uint64_t key; float v; };
        auto locate = [&](int f, Loc& c) {
            int ic = 0, hi = c_in;   // the last ic with cpre[ic] <= f (binary search, warp-uniform)
            while (hi - ic > 1) {
                const int mid = (ic + hi) >> 1;
                if (cpre[mid] <= f) ic = mid; else hi = mid;
            }
            const int s = ((f - cpre[ic]) << 5) + lane;
            c.ic = ic;
            c.xi = -1;
            c.e = -1;
            int pre = 0;
            for (int xi = 0; xi < t.TX; ++xi) {
                const uint32_t lo = rng[2 * (ic * t.TX + xi)], hi = rng[2 * (ic * t.TX + xi) + 1];
                const int n = (int)(hi - lo);
                if (s >= pre && s < pre + n) {
                    c.e = (int64_t)lo + (s - pre);
                    c.xi = xi;
                }
                pre += n;
            }
            c.key = c.e >= 0 ? xkeys[c.e] : 0ull;
            c.v = c.e >= 0 ? xvals[c.e] : 0.0f;
        };
        // warp w takes a contiguous run of chunks (mostly one input channel): concurrent warps
        // then mostly update different dw words
        const int per = (nchunks + nwarps - 1) / nwarps;
        const int fb = min(nchunks, warp * per), fe = min(nchunks, fb + per);
        Loc first{};
        if (fb < fe) locate(fb, first);
        for (int pp = 0; pp < ocp; ++pp) {
        const int nocp = min(ocs, nocl - pp * ocs);   // channels of this pass
        if (pp > 0) __syncthreads();   // the previous pass's sweep of G is complete
        // "initialize dense buffer with gradients(b, oc)", tile + halo, this oc group:
        // per (oc, halo x-row) the kept outputs of the halo y-range are one contiguous key run
        // the warp's rows r = warp + k * nwarps: lane k loads row k's bounds (one latency for all)
        for (int r0 = warp; r0 < nocp * HWX; r0 += 32 * nwarps) {
            uint32_t be0 = 0, be1 = 0;
            int gb = 0;
            uint32_t rz = 0;
            {
                const int r = r0 + lane * nwarps;
                if (r < nocp * HWX) {
                    const int rg = pp * ocs * HWX + r;   // halo row of the group
                    const int64_t row = halo_row(ig, rg, gb);
                    if (row >= 0) {   // (bounds prefetched with the item)
                        be0 = fbd[2 * rg];
                        be1 = fbd[2 * rg + 1];
                        rz = (uint32_t)((uint64_t)row * (uint64_t)gy.Z);
                    }
                }
            }
            // the rows' entries as one list (row k owns positions cum_k .. cum_k + len_k - 1), eight
            // positions per lane in flight per batch; row starts in the warp's scratch words
            const uint32_t len = be1 - be0;
            const uint32_t incl = warp_incl_scan(len);
            const uint32_t wtot = __shfl_sync(kFull, incl, 31);
            // the non-empty rows, compacted: their starts cum_k are strictly increasing, so the
            // row of list position pos is (rows starting at or before pos) - 1
            const unsigned nzm = __ballot_sync(kFull, len != 0u);
            const int kc = __popc(nzm & ((1u << lane) - 1u));
            __syncwarp();
            if (len != 0u) {
                st_eb[kc] = (int)(incl - len);   // cum_k
                st_eb[32 + kc] = (int)be0;       // e0_k
                st_gb[kc] = gb;
                st_rz[kc] = rz;
            }
            __syncwarp();
            const uint32_t mycum = lane < __popc(nzm) ? (uint32_t)st_eb[lane] : 0xffffffffu;
            for (uint32_t base = 0; base < wtot; base += 256) {
                uint64_t kk[8];
                float dv[8];
                int rk[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t w0 = base + 32u * j;   // window of 32 list positions (warp-uniform)
                    const uint32_t pos = w0 + (uint32_t)lane;
                    rk[j] = -1;
                    kk[j] = 0ull;
                    dv[j] = 0.0f;
                    if (w0 >= wtot) continue;
                    // rows starting at or before w0, plus one bit per row starting inside the window
                    const int before = __popc(__ballot_sync(kFull, mycum <= w0));
                    const uint32_t d = mycum - w0;
                    const uint32_t bits = __reduce_or_sync(kFull, (mycum > w0 && d < 32u) ? (1u << d) : 0u);
                    const int k = before + __popc(bits & (0xffffffffu >> (31 - lane))) - 1;
                    if (pos < wtot) {
                        const uint32_t e = (uint32_t)st_eb[32 + k] + (pos - (uint32_t)st_eb[k]);
                        kk[j] = ykeys[e];
                        dv[j] = dy[e];
                        rk[j] = k;
                    }
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (rk[j] < 0) continue;
                    const int gbase = st_gb[rk[j]];
                    const uint32_t L = (uint32_t)kk[j] - st_rz[rk[j]];   // offset in the halo rows (mod 2^32)
                    uint32_t yr = __float2uint_rz(__uint2float_rz(L) * invZ);
                    if (yr * (uint32_t)gy.Z > L) --yr;
                    if ((yr + 1) * (uint32_t)gy.Z <= L) ++yr;
                    G[gbase + (int)yr * sY + (int)(L - yr * (uint32_t)gy.Z)] = dv[j];
                }
            }
            __syncwarp();
        }
        __syncthreads();
        Loc cur{}, nxt{};
        if (pp == 0) cur = first;
        else if (fb < fe) locate(fb, cur);
        for (int f = fb; f < fe; ++f) {
            if (f + 1 < fe) locate(f + 1, nxt);
            const int ic = cur.ic;
            const int64_t e = cur.e;
            int eb = eb_safe;
            const float v = cur.v;
            if (e >= 0) {
                const int64_t r0 = (((ig.b * c_in + ic) * gx.W + ig.wp) * gx.X + ig.x0 + cur.xi) * (int64_t)gx.Y + ig.y0;
                const uint32_t L = (uint32_t)(cur.key - (uint64_t)r0 * (uint64_t)gx.Z);
                const uint32_t yl = div_small(L, (uint32_t)gx.Z, invXZ);   // L < TY * Z
                const int z = (int)(L - yl * (uint32_t)gx.Z);
                eb = kg.hw * sW + (cur.xi + kg.hx) * sX + ((int)yl + kg.hy) * sY + z + kg.hz;
            }
            __syncwarp();
            st_eb[lane] = eb * (int)sizeof(float);   // byte offsets into G
            st_v[lane] = v;
            __syncwarp();
            const int n = lbase[pp * (c_in + 1) + ic + 1] - lbase[pp * (c_in + 1) + ic];
            const int lb = lbase[pp * (c_in + 1) + ic];
            const char* Gb = reinterpret_cast<const char*>(G);
            float prod[32];
#pragma unroll
            for (int q = 0; q < 32; ++q) prod[q] = 0.0f;
            // four 32-weight blocks per sweep over the 32 staged entries: each entry's staged
            // (G offset, value) is read once per sweep instead of once per block
            constexpr int NB = 4;
            for (int wb = 0; wb < n; wb += 32 * NB) {
                int wd[NB];
                float wl[NB], dwl[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    const int j = wb + 32 * b + lane;
                    const bool wok = j < n;
                    wd[b] = (wok ? wdel[lb + j] : wdel[lb]) * (int)sizeof(float);
                    wl[b] = wok ? wv[lb + j] : 0.0f;
                    dwl[b] = 0.0f;
                }
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const int ebq = st_eb[q];
                    const float vq = st_v[q];
#pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        const float g = *reinterpret_cast<const float*>(Gb + (ebq - wd[b]));
                        prod[q] = fmaf(g, wl[b], prod[q]);     // bp_data contribution
                        dwl[b] = fmaf(g, vq, dwl[b]);          // bp_filter contribution
                    }
                }
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    const int j = wb + 32 * b + lane;
                    if (DW && j < n && dwl[b] != 0.0f) atomicAdd(&dwp[lb + j], (double)dwl[b]);
                }
            }
            float dxa = 0.0f;
            if (DX) dxa = reduce_scatter32(prod, lane);   // lane e: sum over this ic's weights
            if (DX && e >= 0) {
                // the same lane owns entry e in every pass (same chunk split): plain
                // read-modify-write of its own earlier pass, atomics only across CTAs
                if (t.n_ocg > 1) atomicAdd(&dx[e], dxa);
                else if (pp == 0) dx[e] = dxa;
                else dx[e] += dxa;
            }
            __syncwarp();
            cur = nxt;
        }
        __syncthreads();
        // zero G for the next item: one vectorized sweep of the slab (a few hundred warp
        // instructions) instead of revisiting every scattered gradient
        {
            float4* G4 = reinterpret_cast<float4*>(G);
            const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
            for (int i = threadIdx.x; i < (gsize >> 2); i += THREADS) G4[i] = z4;
            for (int i = (gsize & ~3) + threadIdx.x; i < gsize; i += blockDim.x) G[i] = 0.0f;
        }
        }   // passes
    }
    __syncthreads();
    if (DW) {   // slot j of a range is table entry t0 + j
        for (int q = warp; q < c_in * ocp; q += nwarps) {
            const int pp = q / c_in, ic = q - pp * c_in;
            const int lb = lbase[pp * (c_in + 1) + ic], t0 = wo(pp, ic), n = wo(pp + 1, ic) - t0;
            for (int j = lane; j < n; j += 32) {
                const double v = dwp[lb + j];
                if (v != 0.0) atomicAdd(&dw_acc[wsrc[t0 + j]], v);
            }
        }
    }
}

template <bool DX, bool DW, int THREADS>
static cudaError_t launch_bwd_tt(const Geo& gx, const Geo& gy, const KGeo& kg, const BwdTile& t,
                                Keys xkeys, const float* xvals, const uint32_t* xrow,
                                Keys ykeys, const float* dy, const uint32_t* yrow,
                                const int2* wmeta, const float* wval, const int* woff, const int* wsrc,
                                float* dx, double* dw_acc, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(conv_bwd_kernel<DX, DW, THREADS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t.smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)t.grid, (unsigned)t.n_ocg);
    { SPC_PHASE("conv_bwd", s, 1); conv_bwd_kernel<DX, DW, THREADS><<<grid, THREADS, t.smem, s>>>(
          gx, gy, kg, t, xkeys, xvals, xrow, ykeys, dy, yrow, wmeta, wval, woff, wsrc, dx, dw_acc); }
    return cudaGetLastError();
}

template <bool DX, bool DW>
static cudaError_t launch_bwd_t(const Geo& gx, const Geo& gy, const KGeo& kg, const BwdTile& t,
                                Keys xkeys, const float* xvals, const uint32_t* xrow,
                                Keys ykeys, const float* dy, const uint32_t* yrow,
                                const int2* wmeta, const float* wval, const int* woff, const int* wsrc,
                                float* dx, double* dw_acc, cudaStream_t s) {
    if (t.threads == 256)
        return launch_bwd_tt<DX, DW, 256>(gx, gy, kg, t, xkeys, xvals, xrow, ykeys, dy, yrow, wmeta, wval, woff, wsrc,
                                          dx, dw_acc, s);
    return launch_bwd_tt<DX, DW, 512>(gx, gy, kg, t, xkeys, xvals, xrow, ykeys, dy, yrow, wmeta, wval, woff, wsrc,
                                      dx, dw_acc, s);
}

cudaError_t launch_conv_bwd(const Geo& gx, const Geo& gy, const KGeo& kg, const BwdTile& t,
                            Keys xkeys, const float* xvals, const uint32_t* xrow,
                            Keys ykeys, const float* dy, const uint32_t* yrow,
                            const int2* wmeta, const float* wval, const int* woff, const int* wsrc,
                            float* dx, double* dw_acc, bool want_dx, bool want_dw, cudaStream_t s) {
    if (gx.B == 0) return cudaSuccess;
    {
        SPC_PHASE("bwd_slot_order", s, 1);
        bwd_slot_order_kernel<<<(unsigned)t.n_ocg, 512, 0, s>>>(kg, t, (int)gx.C, (int)gy.C, const_cast<int2*>(wmeta),
                                                                 const_cast<float*>(wval), const_cast<int*>(wsrc), woff);
    }
    if (want_dx && want_dw)
        return launch_bwd_t<true, true>(gx, gy, kg, t, xkeys, xvals, xrow, ykeys, dy, yrow, wmeta, wval, woff, wsrc,
                                        dx, dw_acc, s);
    if (want_dx)
        return launch_bwd_t<true, false>(gx, gy, kg, t, xkeys, xvals, xrow, ykeys, dy, yrow, wmeta, wval, woff,
                                         wsrc, dx, dw_acc, s);
    return launch_bwd_t<false, true>(gx, gy, kg, t, xkeys, xvals, xrow, ykeys, dy, yrow, wmeta, wval, woff, wsrc,
                                     dx, dw_acc, s);
}

// dbias[oc] = sum of dy over the kept outputs of oc (fp64), reading R13. Segment (b, oc) owns
// the contiguous entry range yrow[s*R] .. yrow[(s+1)*R] of the row index, so a block sums a
// slice of one segment with coalesced loads and adds it to dbias[oc] once.
__global__ void __launch_bounds__(256) dbias_kernel(Geo gy, const uint32_t* __restrict__ yrow,
                                                    const float* __restrict__ dy, int splits,
                                                    double* __restrict__ db) {
    __shared__ double sm[33];
    const int64_t s = blockIdx.x / splits;
    const int j = blockIdx.x - (int)(s * splits);
    const int64_t e0 = yrow[s * gy.R], e1 = yrow[(s + 1) * gy.R];
    const int64_t len = e1 - e0, per = (len + splits - 1) / splits;
    const int64_t lo = e0 + j * per, hi = min(e1, lo + per);
    double acc = 0.0;
    for (int64_t t = lo + threadIdx.x; t < hi; t += blockDim.x) acc += (double)dy[t];
    acc = block_sum(acc, sm);
    if (threadIdx.x == 0 && acc != 0.0) atomicAdd(&db[s % gy.C], acc);
}

cudaError_t launch_dbias(const Geo& gy, const uint32_t* yrow, const float* dy, double* db_acc, cudaStream_t s) {
    const int64_t nseg = gy.B * gy.C;
    if (nseg <= 0) return cudaSuccess;
    const int splits = (int)std::max<int64_t>(1, std::min<int64_t>(64, (4 * num_sms() + nseg - 1) / nseg));
    { SPC_PHASE("dbias", s, 1); dbias_kernel<<<(unsigned)(nseg * splits), 256, 0, s>>>(gy, yrow, dy, splits, db_acc); }
    return cudaGetLastError();
}

}  // namespace spc

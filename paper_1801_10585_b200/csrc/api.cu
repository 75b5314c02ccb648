// C-ABI entry points of libspconv (include/spconv.h): argument validation, workspace carving
// and kernel launches. No device memory is allocated here; every buffer is the caller's.
#include "spc_internal.cuh"

#include <stdlib.h>
#include <string.h>
#include <algorithm>
#include <cmath>

using namespace spc;

namespace {

constexpr size_t kAlign = 256;

// Carves a caller-provided workspace; with base == nullptr it only measures.
struct Carver {
    char* base;
    size_t used = 0;
    explicit Carver(void* b) : base(static_cast<char*>(b)) {}
    template <typename T>
    T* take(size_t count) {
        used = (used + kAlign - 1) & ~(kAlign - 1);
        T* p = base ? reinterpret_cast<T*>(base + used) : nullptr;
        used += sizeof(T) * (count ? count : 1);
        return p;
    }
};

bool validate_env() {
    const char* v = getenv("SPC_VALIDATE");
    return v && v[0] == '1';
}

spc_status_t check_map(const spc_map_t* m, bool need_values = true) {
    if (!m) return SPC_ERR_INVALID_ARG;
    if (m->ndim < 1 || m->ndim > SPC_MAX_NDIM) return SPC_ERR_UNSUPPORTED;
    if (m->batch < 0 || m->channels < 1 || m->nnz < 0) return SPC_ERR_SHAPE;
    double total = (double)m->batch * (double)m->channels;
    for (int d = 0; d < m->ndim; ++d) {
        if (m->dims[d] < 1 || m->dims[d] > (1ll << 30)) return SPC_ERR_SHAPE;
        total *= (double)m->dims[d];
    }
    if (total >= 9.2e18) return SPC_ERR_SHAPE;
    if (m->nnz >= (1ll << 32) - 1) return SPC_ERR_UNSUPPORTED;   // 32-bit row index
    if (m->nnz > 0 && (!m->keys || (need_values && !m->values))) return SPC_ERR_INVALID_ARG;
    if (m->key_bits != 0 && m->key_bits != 32 && m->key_bits != 64) return SPC_ERR_INVALID_ARG;
    if (m->key_bits == 32 && total > 4294967296.0) return SPC_ERR_UNSUPPORTED;   // keys must fit 32 bits
    return SPC_OK;
}

Geo geo_of(const spc_map_t* m, int64_t channels) {
    Geo g{};
    int64_t d[4] = {1, 1, 1, 1};
    for (int i = 0; i < m->ndim; ++i) d[4 - m->ndim + i] = m->dims[i];
    g.B = m->batch;
    g.C = channels;
    g.W = (int)d[0];
    g.X = (int)d[1];
    g.Y = (int)d[2];
    g.Z = (int)d[3];
    g.V = d[0] * d[1] * d[2] * d[3];
    g.R = d[0] * d[1] * d[2];
    return g;
}

spc_status_t check_filter(const spc_filter_t* w, const spc_map_t* x, KGeo* kg) {
    if (!w) return SPC_ERR_INVALID_ARG;
    if (w->ndim != x->ndim) return SPC_ERR_SHAPE;
    if (w->c_in != x->channels || w->c_out < 1 || w->nnz < 0) return SPC_ERR_SHAPE;
    if (w->c_in * w->c_out > (1ll << 28)) return SPC_ERR_UNSUPPORTED;
    int64_t k[4] = {1, 1, 1, 1};
    int64_t kv = 1;
    for (int i = 0; i < w->ndim; ++i) {
        if (w->ksize[i] < 1 || w->ksize[i] % 2 == 0) return SPC_ERR_SHAPE;
        k[4 - w->ndim + i] = w->ksize[i];
        kv *= w->ksize[i];
    }
    if (kv > 1024) return SPC_ERR_UNSUPPORTED;
    if (w->ndim == 4 && w->c_out >= (1 << 21)) return SPC_ERR_UNSUPPORTED;   // meta packing (pack_oc_ow)
    if (w->nnz > w->c_in * w->c_out * kv) return SPC_ERR_SHAPE;
    if (w->nnz > 0 && (!w->keys || !w->values)) return SPC_ERR_INVALID_ARG;
    kg->kw = (int)k[0]; kg->kx = (int)k[1]; kg->ky = (int)k[2]; kg->kz = (int)k[3];
    kg->hw = kg->kw / 2; kg->hx = kg->kx / 2; kg->hy = kg->ky / 2; kg->hz = kg->kz / 2;
    kg->KV = (int)kv;
    return SPC_OK;
}

// space: the output map's batch*channels*prod(dims) (its keys must fit 32 bits when key_bits = 32)
spc_status_t check_out(const spc_map_out_t* y, int64_t need, double space = 0.0) {
    if (!y) return SPC_ERR_INVALID_ARG;
    if (!y->nnz_dev) return SPC_ERR_INVALID_ARG;
    if (y->capacity < need) return SPC_ERR_CAPACITY;
    if (need > 0 && (!y->keys || !y->values)) return SPC_ERR_INVALID_ARG;
    if (y->key_bits != 0 && y->key_bits != 32 && y->key_bits != 64) return SPC_ERR_INVALID_ARG;
    if (y->key_bits == 32 && space > 4294967296.0) return SPC_ERR_UNSUPPORTED;
    return SPC_OK;
}

double space_of(const spc_map_t* m, int64_t channels) {
    double v = (double)m->batch * (double)channels;
    for (int d = 0; d < m->ndim; ++d) v *= (double)m->dims[d];
    return v;
}

spc_status_t cu(cudaError_t e) { return e == cudaSuccess ? SPC_OK : SPC_ERR_CUDA; }

// key arrays of either width (spc_map_t::key_bits, Table 1 "Sparse 32")
Keys kin(const spc_map_t* m) { return Keys(m->keys, m->key_bits == 32); }
KeysOut kout(const spc_map_out_t* y) { return KeysOut(y->keys, y->key_bits == 32); }

#define SPC_TRY(expr)                          \
    do {                                       \
        spc_status_t _s = (expr);              \
        if (_s != SPC_OK) return _s;           \
    } while (0)

// SPC_VALIDATE=1: device check of sortedness and range; synchronises the stream.
spc_status_t maybe_validate(const spc_map_t* m, int* flag, cudaStream_t s) {
    if (!flag) return SPC_OK;
    uint64_t limit = (uint64_t)m->batch * (uint64_t)m->channels;
    for (int d = 0; d < m->ndim; ++d) limit *= (uint64_t)m->dims[d];
    SPC_TRY(cu(cudaMemsetAsync(flag, 0, sizeof(int), s)));
    SPC_TRY(cu(launch_validate(kin(m), m->nnz_dev, m->nnz, limit, flag, s)));
    int h = 0;
    SPC_TRY(cu(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s)));
    SPC_TRY(cu(cudaStreamSynchronize(s)));
    return h ? SPC_ERR_UNSORTED : SPC_OK;
}

// SPC_VALIDATE=1: the filter keys too -- strictly increasing, below c_out*c_in*prod(ksize)
// (an unsorted, duplicated or out-of-range filter would otherwise index the filter tables out of
// bounds). Synchronises the stream.
spc_status_t maybe_validate_filter(const spc_filter_t* w, int* flag, cudaStream_t s) {
    if (!flag || w->nnz == 0) return SPC_OK;
    uint64_t kv = 1;
    for (int d = 0; d < w->ndim; ++d) kv *= (uint64_t)w->ksize[d];
    const uint64_t limit = (uint64_t)w->c_out * (uint64_t)w->c_in * kv;
    SPC_TRY(cu(cudaMemsetAsync(flag, 0, sizeof(int), s)));
    SPC_TRY(cu(launch_validate(w->keys, nullptr, w->nnz, limit, flag, s)));
    int h = 0;
    SPC_TRY(cu(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s)));
    SPC_TRY(cu(cudaStreamSynchronize(s)));
    return h ? SPC_ERR_UNSORTED : SPC_OK;
}

struct FilterWs {
    int2* meta;
    float* val;
    int* off;
    int* src;
    int* scratch;
};

FilterWs carve_filter(Carver& c, const spc_filter_t* w) {
    FilterWs f{};
    f.meta = c.take<int2>((size_t)w->nnz);
    f.val = c.take<float>((size_t)w->nnz);
    f.off = c.take<int>((size_t)w->c_in * (w->c_out + 1));
    f.src = c.take<int>((size_t)w->nnz);
    f.scratch = c.take<int>((size_t)2 * w->c_in * w->c_out);
    return f;
}

// ----------------------------------------------------------------------- forward
struct FwdWs {
    GemmArgs g;        // variant G buffers (null unless the variant is G)
    uint32_t* xrow;
    int2* meta2;
    float* val2;
    int* off2;
    int* scratch2;
    FwdArgs a;
    int* flag;
};

// Estimated seconds of the two accumulate variants (AUTO's choice; the Python layer's per-layer
// autotuner replaces it with a measurement). S: Eq. (1) pairs at the measured scatter rate. G:
// per 128-voxel tile and filter offset, the larger of the operand gather (shared-memory bytes at
// 128 B/clk) and the 3xTF32 MMAs (128*N/256 clk per K step), plus the densify traffic.
double est_scatter_s(const spc_map_t* x, const spc_filter_t* w) {
    const double pairs = (double)x->nnz * (double)w->nnz / (double)std::max<int64_t>(1, w->c_in);
    return pairs / 4e11;
}
double est_gemm_s(const Geo& gx, const GemmPlan& g) {
    const double gather = (2.0 * 128 * g.Kp * 4 + 2.0 * g.Np * g.Kp * 4) / 128.0;
    const double mma = 3.0 * (g.Kp / 8) * (128.0 * g.Np / 256.0);
    const double tiles = (double)gx.B * (double)g.ntile;
    return tiles * g.KV * std::max(gather, mma) / ((double)num_sms() * sm_clock_hz()) + (double)gx.B * gx.V * g.Kp * 16.0 / 3e12;
}

spc_status_t fwd_plan(const spc_map_t* x, const spc_filter_t* w, spc_attn_t attn, int64_t k, spc_variant_t variant,
                      Geo* gx, Geo* gy, KGeo* kg, FwdTile* t, GemmPlan* gp, int64_t* cap, int* use_gemm) {
    SPC_TRY(check_map(x));
    SPC_TRY(check_filter(w, x, kg));
    if (attn != SPC_ATTN_NONE && attn != SPC_ATTN_MAGNITUDE && attn != SPC_ATTN_RAW) return SPC_ERR_INVALID_ARG;
    if (attn != SPC_ATTN_NONE && k < 1) return SPC_ERR_INVALID_ARG;
    if (variant != SPC_VARIANT_AUTO && variant != SPC_VARIANT_SCATTER && variant != SPC_VARIANT_GEMM)
        return SPC_ERR_INVALID_ARG;
    *gx = geo_of(x, x->channels);
    *gy = geo_of(x, w->c_out);
    const int64_t per = attn != SPC_ATTN_NONE ? std::min<int64_t>(k, gy->V) : gy->V;
    *cap = x->batch * w->c_out * per;
    const double cells = (double)x->batch * (double)x->channels * (double)gx->V;
    *t = plan_fwd_tile(*gy, *kg, (int)w->c_out, (int)w->c_in, w->nnz, cells > 0 ? (double)x->nnz / cells : 0.0);
    *gp = plan_gemm(*gx, *gy, *kg);
    const bool s_ok = t->smem != 0, g_ok = gp->ok != 0;
    if (variant == SPC_VARIANT_SCATTER) *use_gemm = 0;
    else if (variant == SPC_VARIANT_GEMM) *use_gemm = 1;
    else *use_gemm = g_ok && (!s_ok || est_gemm_s(*gx, *gp) < est_scatter_s(x, w));
    if (*use_gemm ? !g_ok : !s_ok) return SPC_ERR_UNSUPPORTED;
    return SPC_OK;
}

// Candidate capacity: the threshold bucket of a segment holds at most its whole support, so the
// worst case is nseg*V entries (binary data with massive ties); typical use is ~1-2% of that.
FwdWs carve_fwd(Carver& c, const Geo& gx, const Geo& gy, const KGeo& kg, const FwdTile& t, const spc_filter_t* w,
                spc_attn_t attn, const GemmPlan* gp = nullptr) {
    FwdWs ws{};
    if (gp) {
        const size_t nvox = (size_t)(gx.B * gx.V);
        ws.g.xhi = c.take<float>(nvox * gp->Kp);
        ws.g.xlo = c.take<float>(nvox * gp->Kp);
        ws.g.occ = c.take<uint32_t>(nvox);
        ws.g.bhi = c.take<float>((size_t)2 * gp->KV * gp->Np * gp->Kp);   // [W_hi ; W_lo] per offset
        ws.g.blo = nullptr;
        ws.g.wmask = c.take<uint32_t>((size_t)gp->KV * gp->Np);
        ws.g.dinfo = c.take<int>((size_t)3 * gp->KV + 1);
    }
    const int64_t nseg = gy.B * gy.C;
    const size_t KXY = (size_t)kg.kw * kg.kx * kg.ky;
    ws.xrow = c.take<uint32_t>((size_t)(gx.B * gx.C * gx.R + 1));
    ws.meta2 = c.take<int2>((size_t)w->nnz);
    ws.val2 = c.take<float>((size_t)w->nnz);
    ws.off2 = c.take<int>((size_t)w->c_in * KXY * (w->c_out + 1));
    ws.scratch2 = c.take<int>((size_t)2 * w->c_in * KXY * w->c_out);
    FwdArgs& a = ws.a;
    a.seg_count = c.take<unsigned long long>((size_t)nseg);
    a.seg = c.take<FwdSeg>((size_t)nseg);
    a.nseg = nseg;
    a.seg_off = c.take<uint64_t>((size_t)nseg + 1);
    a.cand_cnt = c.take<uint64_t>((size_t)nseg + 1);
    a.cand_cur = c.take<unsigned long long>((size_t)nseg);
    a.seg_stride = (int)gy.C;
    if (gp) {   // variant G: the dense pre-attention buffer and the classify / resolve lists
        a.hist = c.take<uint32_t>((size_t)nseg * kSelBins);
        a.nchunk = (gy.V + 4095) / 4096;
        a.pre = c.take<float>((size_t)(nseg * gy.V));
        a.tile_def = c.take<uint32_t>((size_t)(nseg * a.nchunk));
        a.tile_sel = c.take<uint32_t>((size_t)(nseg * a.nchunk));
        a.tile_off = c.take<uint64_t>((size_t)(nseg * a.nchunk));
        a.cand_off = c.take<uint64_t>((size_t)nseg + 1);
        a.cand = c.take<uint2>(attn == SPC_ATTN_NONE ? 1 : (size_t)(nseg * gy.V));
        a.stg = c.take<uint2>((size_t)(nseg * gy.V));
        a.stg_cnt = c.take<uint64_t>((size_t)nseg + 1);
        a.stg_off = c.take<uint64_t>((size_t)nseg + 1);
        a.stg_cur = c.take<unsigned long long>((size_t)nseg);
        a.chunk_stg = c.take<uint64_t>((size_t)(nseg * a.nchunk));
        a.chunk_ge = c.take<uint32_t>((size_t)(nseg * a.nchunk));
    } else {    // variant S, streamed: candidate runs (8 B per voxel and output channel) + tiles
        plan_fwd_sampling(gy, t, attn, &a);
        const size_t nt = (size_t)nseg * (size_t)a.ntile;
        if (a.nsamp > 0) a.hist = c.take<uint32_t>((size_t)nseg * kSelBins);
        // fewer segments than SMs: the resolve's candidate histogram is split over several CTAs
        // per segment (stream_resolve_hist_kernel) instead of one CTA reading the whole segment
        if (attn != SPC_ATTN_NONE && nseg < num_sms()) {
            a.rhist = c.take<uint32_t>((size_t)nseg * kSelBins);
            a.rstate = c.take<ResolveState>((size_t)nseg);
            a.rsurv = c.take<uint64_t>((size_t)nseg * 4096);
            a.rsurv_n = c.take<uint32_t>((size_t)nseg);
        }
        a.tlow = c.take<uint32_t>((size_t)nseg);
        a.cmax = c.take<uint32_t>((size_t)nseg);
        a.fail = c.take<int>((size_t)nseg);
        a.bflag = c.take<int>((size_t)std::max<int64_t>(gy.B, 1));
        a.redo_b = c.take<int>((size_t)std::max<int64_t>(gy.B, 1));
        a.redo_n = c.take<int>(1);
        a.cpos = c.take<uint32_t>((size_t)(nseg * gy.V));
        a.cval = c.take<float>((size_t)(nseg * gy.V));
        a.tcnt = c.take<uint32_t>(nt);
        a.tile_def = c.take<uint32_t>(nt);
        a.tile_sel = c.take<uint32_t>(nt);
        a.tile_off = c.take<uint64_t>(nt);
    }
    const size_t PK = (size_t)w->c_in * kg.kw * kg.kx;
    a.rnd = c.take<int2>((size_t)t.n_ocg * t.nwg_max + 1);
    a.roff = c.take<int>((size_t)t.n_ocg * (t.ocg * PK + 1));
    a.guard = c.take<int>(1);
    ws.flag = c.take<int>(1);
    return ws;
}

// ---------------------------------------------------------------------- backward
struct BwdWs {
    uint32_t* xrow;
    uint32_t* yrow;
    FilterWs f;
    double* dw_acc;
    double* db_acc;
    int* flag;
};

spc_status_t bwd_plan(const spc_map_t* x, const spc_filter_t* w, const spc_map_t* y, Geo* gx, Geo* gy, KGeo* kg,
                      BwdTile* t) {
    SPC_TRY(check_map(x));
    SPC_TRY(check_map(y, false));
    SPC_TRY(check_filter(w, x, kg));
    if (y->ndim != x->ndim || y->batch != x->batch || y->channels != w->c_out) return SPC_ERR_SHAPE;
    for (int d = 0; d < x->ndim; ++d)
        if (y->dims[d] != x->dims[d]) return SPC_ERR_SHAPE;
    *gx = geo_of(x, x->channels);
    *gy = geo_of(y, y->channels);
    *t = plan_bwd_tile(*gx, *kg, (int)w->c_out, (int)std::min<int64_t>(w->nnz, 1ll << 30));
    if (t->smem == 0) return SPC_ERR_UNSUPPORTED;
    return SPC_OK;
}

BwdWs carve_bwd(Carver& c, const Geo& gx, const Geo& gy, const spc_filter_t* w) {
    BwdWs ws{};
    ws.xrow = c.take<uint32_t>((size_t)(gx.B * gx.C * gx.R + 1));
    ws.yrow = c.take<uint32_t>((size_t)(gy.B * gy.C * gy.R + 1));
    ws.f = carve_filter(c, w);
    ws.dw_acc = c.take<double>((size_t)w->nnz);
    ws.db_acc = c.take<double>((size_t)w->c_out);
    ws.flag = c.take<int>(1);
    return ws;
}

// dw64 / db64 (optional): accumulate into the caller's fp64 buffers and do not round (the
// data-parallel form); otherwise the workspace accumulators are rounded into dw / dbias.
spc_status_t conv_bwd_impl(const spc_map_t* x, const spc_filter_t* w, const spc_map_t* y, const float* dy, float* dx,
                           float* dw, float* dbias, void* workspace, size_t ws_bytes, cudaStream_t s,
                           double* dw64 = nullptr, double* db64 = nullptr) {
    Geo gx, gy;
    KGeo kg;
    BwdTile t;
    SPC_TRY(bwd_plan(x, w, y, &gx, &gy, &kg, &t));
    const bool want_dx = dx != nullptr, want_dw = dw != nullptr || dw64 != nullptr;
    if (y->nnz > 0 && !dy) return SPC_ERR_INVALID_ARG;
    if (!want_dx && !want_dw && !dbias && !db64) return SPC_OK;
    if (want_dx && x->nnz > 0 && !dx) return SPC_ERR_INVALID_ARG;
    Carver m(nullptr);
    carve_bwd(m, gx, gy, w);
    if (!workspace || ws_bytes < m.used) return SPC_ERR_WORKSPACE;
    Carver c(workspace);
    BwdWs ws = carve_bwd(c, gx, gy, w);
    if (validate_env()) {
        SPC_TRY(maybe_validate(x, ws.flag, s));
        SPC_TRY(maybe_validate(y, ws.flag, s));
        SPC_TRY(maybe_validate_filter(w, ws.flag, s));
    }
    if (dw64) ws.dw_acc = dw64;
    if (db64) ws.db_acc = db64;
    SPC_TRY(cu(launch_row_index(gy, kin(y), y->nnz_dev, y->nnz, ws.yrow, s)));
    if (dbias || db64) {
        SPC_TRY(cu(cudaMemsetAsync(ws.db_acc, 0, sizeof(double) * (size_t)w->c_out, s)));
        SPC_TRY(cu(launch_dbias(gy, ws.yrow, dy, ws.db_acc, s)));
    }
    const int64_t nb = (dbias && !db64) ? w->c_out : 0;   // dbias rounded with dw (one launch)
    if (!want_dx && !want_dw) return nb ? cu(launch_f64_to_f32_2(ws.db_acc, dbias, nb, nullptr, nullptr, 0, s)) : SPC_OK;
    SPC_TRY(cu(launch_row_index(gx, kin(x), x->nnz_dev, x->nnz, ws.xrow, s)));
    SPC_TRY(cu(launch_filter_table(kg, (int)w->c_in, (int)w->c_out, w->keys, w->values, w->nnz, ws.f.meta, ws.f.val,
                                   ws.f.off, ws.f.src, ws.f.scratch, s)));
    if (want_dx && t.n_ocg > 1 && x->nnz > 0) SPC_TRY(cu(cudaMemsetAsync(dx, 0, sizeof(float) * (size_t)x->nnz, s)));
    if (want_dw && w->nnz > 0) SPC_TRY(cu(cudaMemsetAsync(ws.dw_acc, 0, sizeof(double) * (size_t)w->nnz, s)));
    SPC_TRY(cu(launch_conv_bwd(gx, gy, kg, t, kin(x), x->values, ws.xrow, kin(y), dy, ws.yrow, ws.f.meta, ws.f.val,
                               ws.f.off, ws.f.src, dx, ws.dw_acc, want_dx, want_dw, s)));
    const int64_t nw = (want_dw && !dw64) ? w->nnz : 0;
    if (nb == 0 && nw == 0) return cu(cudaGetLastError());
    return cu(launch_f64_to_f32_2(ws.db_acc, dbias, nb, ws.dw_acc, dw, nw, s));
}

// -------------------------------------------------------------------- selection ws
struct TopkWs {
    uint32_t* xrow;
    TopkBufs b;
    int* flag;
};

TopkWs carve_topk(Carver& c, const Geo& g, int64_t nnz) {
    TopkWs ws{};
    const int64_t nseg = g.B * g.C;
    const size_t tiles = topk_tiles_bound(nnz, nseg);
    ws.xrow = c.take<uint32_t>((size_t)nseg + 1);   // segment bounds only (no row index)
    ws.b.seg_off = c.take<uint64_t>((size_t)nseg + 1);
    ws.b.tile_start = c.take<uint32_t>((size_t)nseg + 1);
    ws.b.hist = c.take<uint32_t>((size_t)nseg << topk_bits(nnz, nseg));
    ws.b.seg = reinterpret_cast<TkSeg*>(c.take<uint64_t>((size_t)nseg * (topk_seg_bytes() / 8)));
    ws.b.cand_cnt = c.take<uint32_t>((size_t)nseg);
    ws.b.cand = c.take<uint64_t>((size_t)std::max<int64_t>(nnz, 1));
    ws.b.tile_seg = c.take<uint32_t>(tiles);
    ws.b.tile_def = c.take<uint32_t>(tiles);
    ws.b.tile_sel = c.take<uint32_t>(tiles);
    ws.b.tile_off = c.take<uint64_t>(tiles);
    ws.flag = c.take<int>(1);
    return ws;
}

struct ReluWs {
    uint32_t* cnt;
    uint64_t* off;
    uint64_t* tmp;
    int* flag;
};
constexpr int kReluChunkHost = 4096;

ReluWs carve_relu(Carver& c, int64_t n) {
    ReluWs ws{};
    const int64_t nch = std::max<int64_t>(1, (n + kReluChunkHost - 1) / kReluChunkHost);
    ws.cnt = c.take<uint32_t>((size_t)nch);
    ws.off = c.take<uint64_t>((size_t)nch);
    ws.tmp = c.take<uint64_t>(scan_tmp_words(nch));
    ws.flag = c.take<int>(1);
    return ws;
}

struct PoolWs {
    uint32_t* xrow;
    uint32_t* cnt;
    uint64_t* off;
    uint64_t* tmp;
    int* flag;
};

PoolWs carve_pool(Carver& c, const Geo& g, const PoolPlan& p) {
    PoolWs ws{};
    ws.xrow = c.take<uint32_t>(pool_bound_words(g, p));   // band bounds (tile form) or row index
    ws.cnt = c.take<uint32_t>((size_t)p.items);
    ws.off = c.take<uint64_t>((size_t)p.items);
    ws.tmp = c.take<uint64_t>(scan_tmp_words(p.items));
    ws.flag = c.take<int>(1);
    return ws;
}

spc_status_t pool_plan(const spc_map_t* x, const int64_t* stride, Geo* g, PoolPlan* p) {
    SPC_TRY(check_map(x));
    if (!stride) return SPC_ERR_INVALID_ARG;
    int64_t s4[4] = {1, 1, 1, 1};
    for (int i = 0; i < x->ndim; ++i) {
        if (stride[i] < 1 || stride[i] > (1 << 20)) return SPC_ERR_SHAPE;
        s4[4 - x->ndim + i] = stride[i];
    }
    *g = geo_of(x, x->channels);
    *p = plan_pool(*g, (int)s4[0], (int)s4[1], (int)s4[2], (int)s4[3]);
    return SPC_OK;
}

}  // namespace

extern "C" {

const char* spc_version(void) { return "spconv-b200 0.1 (sm_100a)"; }

const char* spc_status_string(spc_status_t s) {
    switch (s) {
        case SPC_OK: return "ok";
        case SPC_ERR_INVALID_ARG: return "invalid argument";
        case SPC_ERR_SHAPE: return "shape mismatch";
        case SPC_ERR_CAPACITY: return "output capacity too small";
        case SPC_ERR_WORKSPACE: return "workspace too small";
        case SPC_ERR_UNSORTED: return "keys unsorted, duplicated or out of range";
        case SPC_ERR_UNSUPPORTED: return "unsupported configuration";
        case SPC_ERR_CUDA: return "CUDA error";
    }
    return "unknown status";
}

spc_status_t spc_conv_fwd_query_ex(const spc_map_t* x, const spc_filter_t* w, spc_attn_t attn, int64_t k,
                                   spc_variant_t variant, int64_t* out_capacity, size_t* workspace_bytes) {
    Geo gx, gy;
    KGeo kg;
    FwdTile t;
    GemmPlan gp;
    int64_t cap;
    int use_gemm;
    SPC_TRY(fwd_plan(x, w, attn, k, variant, &gx, &gy, &kg, &t, &gp, &cap, &use_gemm));
    Carver m(nullptr);
    carve_fwd(m, gx, gy, kg, t, w, attn, use_gemm ? &gp : nullptr);
    if (out_capacity) *out_capacity = cap;
    if (workspace_bytes) *workspace_bytes = m.used;
    return SPC_OK;
}

spc_status_t spc_conv_fwd_query(const spc_map_t* x, const spc_filter_t* w, spc_attn_t attn, int64_t k,
                                int64_t* out_capacity, size_t* workspace_bytes) {
    return spc_conv_fwd_query_ex(x, w, attn, k, SPC_VARIANT_AUTO, out_capacity, workspace_bytes);
}

int spc_conv_fwd_variant(const spc_map_t* x, const spc_filter_t* w, spc_attn_t attn, int64_t k, spc_variant_t variant) {
    Geo gx, gy;
    KGeo kg;
    FwdTile t;
    GemmPlan gp;
    int64_t cap;
    int use_gemm;
    if (fwd_plan(x, w, attn, k, variant, &gx, &gy, &kg, &t, &gp, &cap, &use_gemm) != SPC_OK) return 0;
    return use_gemm ? SPC_VARIANT_GEMM : SPC_VARIANT_SCATTER;
}

spc_status_t sparse_conv_fwd_ex(const spc_map_t* x, const spc_filter_t* w, const float* bias, spc_attn_t attn,
                                int64_t k, spc_variant_t variant, spc_map_out_t* y, void* workspace,
                                size_t workspace_bytes, cudaStream_t s) {
    Geo gx, gy;
    KGeo kg;
    FwdTile t;
    GemmPlan gp;
    int64_t cap;
    int use_gemm;
    SPC_TRY(fwd_plan(x, w, attn, k, variant, &gx, &gy, &kg, &t, &gp, &cap, &use_gemm));
    SPC_TRY(check_out(y, cap, space_of(x, w->c_out)));
    const GemmPlan* gpp = use_gemm ? &gp : nullptr;
    Carver m(nullptr);
    carve_fwd(m, gx, gy, kg, t, w, attn, gpp);
    if (!workspace || workspace_bytes < m.used) return SPC_ERR_WORKSPACE;
    Carver c(workspace);
    FwdWs ws = carve_fwd(c, gx, gy, kg, t, w, attn, gpp);
    if (validate_env()) {
        SPC_TRY(maybe_validate(x, ws.flag, s));
        SPC_TRY(maybe_validate_filter(w, ws.flag, s));
    }
    if (!use_gemm) {   // row index with the value guard fused (the scatter kernel reads the guard)
        SPC_TRY(cu(cudaMemsetAsync(ws.a.guard, 0, sizeof(int), s)));
        SPC_TRY(cu(launch_row_index(gx, kin(x), x->nnz_dev, x->nnz, ws.xrow, s, x->values, ws.a.guard)));
        ws.a.guard_done = 1;
    } else {
        SPC_TRY(cu(launch_row_index(gx, kin(x), x->nnz_dev, x->nnz, ws.xrow, s)));
    }
    if (!use_gemm) {
        SPC_TRY(cu(launch_filter_table_fwd(kg, (int)w->c_in, (int)w->c_out, w->keys, w->values, w->nnz, ws.meta2,
                                           ws.val2, ws.off2, ws.scratch2, s)));
    }
    FwdArgs a = ws.a;
    a.xkeys = kin(x);
    a.x_nnz_dev = x->nnz_dev;
    a.x_nnz = x->nnz;
    a.xvals = x->values;
    a.xrow = ws.xrow;
    a.meta2 = ws.meta2;
    a.val2 = ws.val2;
    a.off2 = ws.off2;
    a.bias = bias;
    a.attn = attn;
    a.k = attn == SPC_ATTN_NONE ? gy.V : k;
    a.out_keys = kout(y);
    a.out_vals = y->values;
    a.out_nnz = y->nnz_dev;
    if (use_gemm) {
        GemmArgs g = ws.g;
        g.xkeys = kin(x);
        g.xvals = x->values;
        g.x_nnz_dev = x->nnz_dev;
        g.x_nnz = x->nnz;
        g.wkeys = w->keys;
        g.wvals = w->values;
        g.nw = w->nnz;
        g.xrow = ws.xrow;
        return cu(launch_conv_fwd_pipeline(gx, gy, kg, t, a, s, &gp, &g));
    }
    return cu(launch_conv_fwd_stream(gx, gy, kg, t, a, s));
}

spc_status_t sparse_conv_fwd(const spc_map_t* x, const spc_filter_t* w, const float* bias, spc_attn_t attn, int64_t k,
                             spc_map_out_t* y, void* workspace, size_t workspace_bytes, cudaStream_t s) {
    return sparse_conv_fwd_ex(x, w, bias, attn, k, SPC_VARIANT_AUTO, y, workspace, workspace_bytes, s);
}

// Batch-sliced forward: the per-(b, oc) workspace -- the pre-attention buffer
// (P:90), candidate and staging lists -- is sized for samples_per_pass samples and reused by
// ceil(batch / samples_per_pass) passes of the scatter pipeline; the outputs of each pass are
// appended in key order (samples are independent in Alg. 1).
spc_status_t spc_conv_fwd_query_pass(const spc_map_t* x, const spc_filter_t* w, spc_attn_t attn, int64_t k,
                                     int64_t samples_per_pass, int64_t* out_capacity, size_t* workspace_bytes) {
    Geo gx, gy;
    KGeo kg;
    FwdTile t;
    GemmPlan gp;
    int64_t cap;
    int use_gemm;
    SPC_TRY(fwd_plan(x, w, attn, k, SPC_VARIANT_SCATTER, &gx, &gy, &kg, &t, &gp, &cap, &use_gemm));
    if (samples_per_pass < 0) return SPC_ERR_INVALID_ARG;
    Geo gyp = gy;
    gyp.B = samples_per_pass == 0 ? gy.B : std::min<int64_t>(samples_per_pass, gy.B);
    Carver m(nullptr);
    carve_fwd(m, gx, gyp, kg, t, w, attn, nullptr);
    if (out_capacity) *out_capacity = cap;
    if (workspace_bytes) *workspace_bytes = m.used;
    return SPC_OK;
}

spc_status_t sparse_conv_fwd_pass(const spc_map_t* x, const spc_filter_t* w, const float* bias, spc_attn_t attn,
                                  int64_t k, int64_t samples_per_pass, spc_map_out_t* y, void* workspace,
                                  size_t workspace_bytes, cudaStream_t s) {
    Geo gx, gy;
    KGeo kg;
    FwdTile t;
    GemmPlan gp;
    int64_t cap;
    int use_gemm;
    SPC_TRY(fwd_plan(x, w, attn, k, SPC_VARIANT_SCATTER, &gx, &gy, &kg, &t, &gp, &cap, &use_gemm));
    if (samples_per_pass < 0) return SPC_ERR_INVALID_ARG;
    SPC_TRY(check_out(y, cap, space_of(x, w->c_out)));
    const int64_t spp = samples_per_pass == 0 ? std::max<int64_t>(gy.B, 1) : std::min<int64_t>(samples_per_pass, std::max<int64_t>(gy.B, 1));
    Geo gyp = gy;
    gyp.B = spp;
    Carver m(nullptr);
    carve_fwd(m, gx, gyp, kg, t, w, attn, nullptr);
    if (!workspace || workspace_bytes < m.used) return SPC_ERR_WORKSPACE;
    Carver c(workspace);
    FwdWs ws = carve_fwd(c, gx, gyp, kg, t, w, attn, nullptr);
    if (validate_env()) {
        SPC_TRY(maybe_validate(x, ws.flag, s));
        SPC_TRY(maybe_validate_filter(w, ws.flag, s));
    }
    SPC_TRY(cu(cudaMemsetAsync(ws.a.guard, 0, sizeof(int), s)));
    SPC_TRY(cu(launch_row_index(gx, kin(x), x->nnz_dev, x->nnz, ws.xrow, s, x->values, ws.a.guard)));
    ws.a.guard_done = 1;
    SPC_TRY(cu(launch_filter_table_fwd(kg, (int)w->c_in, (int)w->c_out, w->keys, w->values, w->nnz, ws.meta2,
                                       ws.val2, ws.off2, ws.scratch2, s)));
    FwdArgs a = ws.a;
    a.xkeys = kin(x);
    a.x_nnz_dev = x->nnz_dev;
    a.x_nnz = x->nnz;
    a.xvals = x->values;
    a.xrow = ws.xrow;
    a.meta2 = ws.meta2;
    a.val2 = ws.val2;
    a.off2 = ws.off2;
    a.bias = bias;
    a.attn = attn;
    a.k = attn == SPC_ATTN_NONE ? gy.V : k;
    a.out_keys = kout(y);
    a.out_vals = y->values;
    a.out_nnz = y->nnz_dev;
    if (gy.B == 0) return cu(cudaMemsetAsync(y->nnz_dev, 0, sizeof(int64_t), s));
    for (int64_t b0 = 0; b0 < gy.B; b0 += spp) {
        Geo gyl = gy;
        gyl.B = std::min<int64_t>(spp, gy.B - b0);
        a.b0 = b0;
        a.seg0 = b0 * gy.C;
        a.nseg = gyl.B * gy.C;
        a.out_append = b0 > 0;
        SPC_TRY(cu(launch_conv_fwd_stream(gx, gyl, kg, t, a, s)));
    }
    return SPC_OK;
}

spc_status_t spc_conv_bwd_query(const spc_map_t* x, const spc_filter_t* w, const spc_map_t* y,
                                size_t* workspace_bytes) {
    Geo gx, gy;
    KGeo kg;
    BwdTile t;
    SPC_TRY(bwd_plan(x, w, y, &gx, &gy, &kg, &t));
    Carver m(nullptr);
    carve_bwd(m, gx, gy, w);
    if (workspace_bytes) *workspace_bytes = m.used;
    return SPC_OK;
}

spc_status_t sparse_conv_bwd(const spc_map_t* x, const spc_filter_t* w, const spc_map_t* y, const float* dy, float* dx,
                             float* dw, float* dbias, void* workspace, size_t workspace_bytes, cudaStream_t s) {
    if (!dx || !dw) return SPC_ERR_INVALID_ARG;
    return conv_bwd_impl(x, w, y, dy, dx, dw, dbias, workspace, workspace_bytes, s);
}

spc_status_t sparse_conv_bwd_input(const spc_map_t* x, const spc_filter_t* w, const spc_map_t* y, const float* dy,
                                   float* dx, void* workspace, size_t workspace_bytes, cudaStream_t s) {
    if (!dx) return SPC_ERR_INVALID_ARG;
    return conv_bwd_impl(x, w, y, dy, dx, nullptr, nullptr, workspace, workspace_bytes, s);
}

spc_status_t sparse_conv_bwd_weight(const spc_map_t* x, const spc_filter_t* w, const spc_map_t* y, const float* dy,
                                    float* dw, float* dbias, void* workspace, size_t workspace_bytes, cudaStream_t s) {
    if (!dw) return SPC_ERR_INVALID_ARG;
    return conv_bwd_impl(x, w, y, dy, nullptr, dw, dbias, workspace, workspace_bytes, s);
}

spc_status_t sparse_conv_bwd_f64(const spc_map_t* x, const spc_filter_t* w, const spc_map_t* y, const float* dy,
                                 float* dx, double* dw64, double* dbias64, void* workspace, size_t workspace_bytes,
                                 cudaStream_t s) {
    if (!dw64) return SPC_ERR_INVALID_ARG;
    return conv_bwd_impl(x, w, y, dy, dx, nullptr, nullptr, workspace, workspace_bytes, s, dw64, dbias64);
}

spc_status_t spc_round_f64(const double* in, float* out, int64_t n, cudaStream_t s) {
    if (n < 0 || (n > 0 && (!in || !out))) return SPC_ERR_INVALID_ARG;
    if (n == 0) return SPC_OK;
    return cu(launch_f64_to_f32(in, out, n, s));
}

spc_status_t spc_topk_query(const spc_map_t* x, spc_attn_t attn, int64_t k, int64_t* out_capacity,
                            size_t* workspace_bytes) {
    SPC_TRY(check_map(x));
    if (attn != SPC_ATTN_MAGNITUDE && attn != SPC_ATTN_RAW) return SPC_ERR_INVALID_ARG;
    if (k < 1) return SPC_ERR_INVALID_ARG;
    const Geo g = geo_of(x, x->channels);
    Carver m(nullptr);
    carve_topk(m, g, x->nnz);
    if (out_capacity) *out_capacity = std::min<int64_t>(x->nnz, g.B * g.C * std::min<int64_t>(k, g.V));
    if (workspace_bytes) *workspace_bytes = m.used;
    return SPC_OK;
}

spc_status_t attention_topk(const spc_map_t* x, spc_attn_t attn, int64_t k, spc_map_out_t* y, int64_t* src_index,
                            void* workspace, size_t workspace_bytes, cudaStream_t s) {
    int64_t cap;
    size_t need;
    SPC_TRY(spc_topk_query(x, attn, k, &cap, &need));
    SPC_TRY(check_out(y, cap, space_of(x, x->channels)));
    if (!workspace || workspace_bytes < need) return SPC_ERR_WORKSPACE;
    const Geo g = geo_of(x, x->channels);
    Carver c(workspace);
    TopkWs ws = carve_topk(c, g, x->nnz);
    if (validate_env()) SPC_TRY(maybe_validate(x, ws.flag, s));
    SPC_TRY(cu(launch_seg_bounds(kin(x), x->nnz_dev, x->nnz, g.B * g.C, g.V, ws.xrow, s)));
    return cu(launch_topk(kin(x), x->values, ws.xrow, g.B * g.C, x->nnz, attn, k, ws.b, kout(y), y->values,
                          src_index, y->nnz_dev, s));
}

spc_status_t spc_relu_query(const spc_map_t* x, int64_t* out_capacity, size_t* workspace_bytes) {
    SPC_TRY(check_map(x));
    Carver m(nullptr);
    carve_relu(m, x->nnz);
    if (out_capacity) *out_capacity = x->nnz;
    if (workspace_bytes) *workspace_bytes = m.used;
    return SPC_OK;
}

spc_status_t sparse_relu(const spc_map_t* x, spc_map_out_t* y, int64_t* src_index, void* workspace,
                         size_t workspace_bytes, cudaStream_t s) {
    int64_t cap;
    size_t need;
    SPC_TRY(spc_relu_query(x, &cap, &need));
    SPC_TRY(check_out(y, cap, space_of(x, x->channels)));
    if (!workspace || workspace_bytes < need) return SPC_ERR_WORKSPACE;
    Carver c(workspace);
    ReluWs ws = carve_relu(c, x->nnz);
    if (validate_env()) SPC_TRY(maybe_validate(x, ws.flag, s));
    return cu(launch_relu(kin(x), x->values, x->nnz_dev, x->nnz, ws.cnt, ws.off, ws.tmp, kout(y), y->values, src_index,
                          y->nnz_dev, s));
}

spc_status_t spc_maxpool_query(const spc_map_t* x, const int64_t* stride, int64_t* out_capacity,
                               size_t* workspace_bytes) {
    Geo g;
    PoolPlan p;
    SPC_TRY(pool_plan(x, stride, &g, &p));
    Carver m(nullptr);
    carve_pool(m, g, p);
    if (out_capacity) *out_capacity = x->nnz;
    if (workspace_bytes) *workspace_bytes = m.used;
    return SPC_OK;
}

spc_status_t sparse_maxpool(const spc_map_t* x, const int64_t* stride, spc_map_out_t* y, int64_t* argmax,
                            void* workspace, size_t workspace_bytes, cudaStream_t s) {
    Geo g;
    PoolPlan p;
    SPC_TRY(pool_plan(x, stride, &g, &p));
    SPC_TRY(check_out(y, x->nnz, space_of(x, x->channels)));
    Carver m(nullptr);
    carve_pool(m, g, p);
    if (!workspace || workspace_bytes < m.used) return SPC_ERR_WORKSPACE;
    Carver c(workspace);
    PoolWs ws = carve_pool(c, g, p);
    if (validate_env()) SPC_TRY(maybe_validate(x, ws.flag, s));
    if (!p.tiled) SPC_TRY(cu(launch_row_index(g, kin(x), x->nnz_dev, x->nnz, ws.xrow, s)));
    return cu(launch_maxpool(g, p, kin(x), x->values, x->nnz_dev, x->nnz, ws.xrow, ws.cnt, ws.off, ws.tmp, kout(y), y->values, argmax,
                             y->nnz_dev, s));
}

spc_status_t sparse_scatter_grad(const int64_t* src_index, const float* dy, int64_t n_out_bound,
                                 const int64_t* n_out_dev, float* dx, int64_t n_in, cudaStream_t s) {
    if (n_out_bound < 0 || n_in < 0) return SPC_ERR_SHAPE;
    if (n_out_bound > 0 && (!src_index || !dy)) return SPC_ERR_INVALID_ARG;
    if (n_in > 0 && !dx) return SPC_ERR_INVALID_ARG;
    if (n_in == 0) return SPC_OK;
    return cu(launch_scatter_grad(src_index, dy, n_out_bound, n_out_dev, dx, n_in, s));
}

spc_status_t sparse_scatter_grad_sorted(const int64_t* src_index, const float* dy, int64_t n_out_bound,
                                        const int64_t* n_out_dev, float* dx, int64_t n_in, cudaStream_t s) {
    if (n_out_bound < 0 || n_in < 0) return SPC_ERR_SHAPE;
    if (n_out_bound > 0 && (!src_index || !dy)) return SPC_ERR_INVALID_ARG;
    if (n_in > 0 && !dx) return SPC_ERR_INVALID_ARG;
    if (n_in == 0) return SPC_OK;
    if (validate_env() && n_out_bound > 0) {   // strictly increasing and in range; synchronises
        int* flag = nullptr;
        SPC_TRY(cu(cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(int), s)));
        int h = 0;
        cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int), s);
        if (e == cudaSuccess) e = launch_check_sorted(src_index, n_out_bound, n_out_dev, n_in, flag, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaFreeAsync(flag, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        SPC_TRY(cu(e));
        if (h) return SPC_ERR_UNSORTED;
    }
    return cu(launch_scatter_grad_sorted(src_index, dy, n_out_bound, n_out_dev, dx, n_in, s));
}

}  // extern "C"

// ------------------------------------------------------------------ training-loop steps (f1)
spc_status_t sparse_adagrad_step(float* params, const float* grad, float* accum, int64_t n, const int64_t* y_nnz_dev,
                                 double y_cells, const spc_density_reg_t* reg, double lr, double eps, cudaStream_t s) {
    if (n < 0 || (n > 0 && (!params || !grad || !accum))) return SPC_ERR_INVALID_ARG;
    if (reg && (!y_nnz_dev || !(y_cells > 0.0))) return SPC_ERR_INVALID_ARG;
    DensityReg r{};
    if (reg) r = DensityReg{reg->lambda, reg->rho_up, reg->o, reg->b1, reg->b2};
    return cu(launch_adagrad(params, grad, accum, n, y_nnz_dev, y_cells, r, reg != nullptr, lr, eps, s));
}

spc_status_t spc_prune_query(int64_t n, size_t* workspace_bytes) {
    if (n < 0) return SPC_ERR_INVALID_ARG;
    if (workspace_bytes) *workspace_bytes = prune_ws_words(n) * sizeof(uint64_t);
    return SPC_OK;
}

spc_status_t sparse_filter_prune(const uint64_t* keys, const float* values, const float* accum, const uint8_t* warn,
                                 int64_t n, double eps, uint64_t* out_keys, float* out_values, float* out_accum,
                                 uint8_t* out_warn, int64_t* out_nnz_dev, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (n < 0 || !out_nnz_dev) return SPC_ERR_INVALID_ARG;
    if (n > 0 && (!keys || !values || !warn || !out_keys || !out_values || !out_warn)) return SPC_ERR_INVALID_ARG;
    if ((accum == nullptr) != (out_accum == nullptr)) return SPC_ERR_INVALID_ARG;
    if (!ws || ws_bytes < prune_ws_words(n) * sizeof(uint64_t)) return SPC_ERR_WORKSPACE;
    return cu(launch_prune(keys, values, accum, warn, n, eps, out_keys, out_values, out_accum, out_warn, out_nnz_dev,
                           static_cast<uint64_t*>(ws), s));
}

// ------------------------------------------------------------------ sparseToDense bridge (f3)
spc_status_t sparse_to_dense(const spc_map_t* x, float* dense, cudaStream_t s) {
    SPC_TRY(check_map(x));
    if (!dense) return SPC_ERR_INVALID_ARG;
    const Geo g = geo_of(x, x->channels);
    return cu(launch_to_dense(kin(x), x->values, x->nnz_dev, x->nnz, dense, g.B * g.C * g.V, s));
}

spc_status_t sparse_to_dense_bwd(const spc_map_t* x, const float* ddense, float* dvalues, cudaStream_t s) {
    SPC_TRY(check_map(x, false));
    if (!ddense || (x->nnz > 0 && !dvalues)) return SPC_ERR_INVALID_ARG;
    return cu(launch_gather_dense(kin(x), x->nnz_dev, x->nnz, ddense, dvalues, s));
}

// ------------------------------------------------------------------ memory model (f2)
extern "C" spc_status_t spc_memory_estimate(int32_t ndim, int64_t r, int64_t batch, int64_t channels, double rho_up,
                                            int32_t index_bits, double* dense_bytes, double* sparse_bytes,
                                            double* temp_bytes) {
    if (ndim < 1 || ndim > SPC_MAX_NDIM || r < 1 || batch < 1 || channels < 1 || !(rho_up > 0.0 && rho_up <= 1.0) ||
        (index_bits != 32 && index_bits != 64))
        return SPC_ERR_INVALID_ARG;
    double cells = 1.0;   // r^k (exact in double up to 2^53)
    for (int d = 0; d < ndim; ++d) cells *= (double)r;
    const double space = cells * (double)batch * (double)channels;
    if (index_bits == 32 && space >= 4294967296.0) return SPC_ERR_UNSUPPORTED;   // App. A
    if (dense_bytes) *dense_bytes = space * 4.0;
    if (sparse_bytes) *sparse_bytes = std::ceil(rho_up * cells) * (double)batch * (double)channels * (index_bits / 8 + 4);
    if (temp_bytes) *temp_bytes = cells * 8.0;
    return SPC_OK;
}

// ------------------------------------------------------------------ 32-bit key storage (f2)
namespace {
bool fits32(const spc_map_t* x) {
    double space = (double)x->batch * (double)x->channels;
    for (int d = 0; d < x->ndim; ++d) space *= (double)x->dims[d];
    return space < 4294967296.0;
}
}  // namespace

// ------------------------------------------------------------------ key codec
static spc_status_t codec_geo(int32_t ndim, int64_t batch, int64_t channels, const int64_t* dims, int64_t n,
                              CodecGeo* g) {
    if (ndim < 1 || ndim > SPC_MAX_NDIM || !dims || n < 0) return SPC_ERR_INVALID_ARG;
    if (batch <= 0 || channels <= 0) return SPC_ERR_SHAPE;
    g->nd = ndim;
    g->B = batch;
    g->C = channels;
    double tot = (double)batch * (double)channels;
    uint64_t V = 1;
    for (int d = 0; d < ndim; ++d) {
        if (dims[d] <= 0) return SPC_ERR_SHAPE;
        g->d[d] = dims[d];
        tot *= (double)dims[d];
        if (tot >= 9.2e18) return SPC_ERR_SHAPE;   // key space above 2^63
        V *= (uint64_t)dims[d];
    }
    g->V = V;
    g->total = (uint64_t)batch * (uint64_t)channels * V;
    return SPC_OK;
}

extern "C" spc_status_t spc_encode_keys(int32_t ndim, int64_t batch, int64_t channels, const int64_t* dims,
                                        const int64_t* coords, int64_t n, uint64_t* keys, int* bad_dev,
                                        cudaStream_t s) {
    CodecGeo g{};
    SPC_TRY(codec_geo(ndim, batch, channels, dims, n, &g));
    if (n > 0 && (!coords || !keys)) return SPC_ERR_INVALID_ARG;
    return cu(launch_encode_keys(g, coords, n, keys, bad_dev, s));
}

extern "C" spc_status_t spc_decode_keys(int32_t ndim, int64_t batch, int64_t channels, const int64_t* dims,
                                        const uint64_t* keys, int64_t n, int64_t* coords, int* bad_dev,
                                        cudaStream_t s) {
    CodecGeo g{};
    SPC_TRY(codec_geo(ndim, batch, channels, dims, n, &g));
    if (n > 0 && (!coords || !keys)) return SPC_ERR_INVALID_ARG;
    return cu(launch_decode_keys(g, keys, n, coords, bad_dev, s));
}

extern "C" spc_status_t sparse_keys_narrow(const spc_map_t* x, uint32_t* keys32, cudaStream_t s) {
    SPC_TRY(check_map(x, false));
    if (x->key_bits == 32) return SPC_ERR_INVALID_ARG;   // already 32-bit
    if (!fits32(x)) return SPC_ERR_UNSUPPORTED;
    if (x->nnz > 0 && !keys32) return SPC_ERR_INVALID_ARG;
    return cu(launch_keys_narrow(x->keys, x->nnz_dev, x->nnz, keys32, s));
}

extern "C" spc_status_t sparse_keys_widen(const uint32_t* keys32, const int64_t* nnz_dev, int64_t nnz, uint64_t* keys,
                                          cudaStream_t s) {
    if (nnz < 0 || (nnz > 0 && (!keys32 || !keys))) return SPC_ERR_INVALID_ARG;
    return cu(launch_keys_widen(keys32, nnz_dev, nnz, keys, s));
}

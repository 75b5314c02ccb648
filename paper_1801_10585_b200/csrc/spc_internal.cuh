// Internal declarations of libspconv (not part of the ABI). sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/spconv.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libspconv is written for sm_100a (B200) only"
#endif

namespace spc {

// Absent marker of the pre-attention accumulators: a signalling-NaN pattern. GPU arithmetic
// only ever produces the canonical quiet NaN 0x7fffffff, so a NaN that arises from the data
// (NaN/Inf inputs, inf - inf) stays a value and propagates instead of being read as "absent".
constexpr uint32_t kAbsent = 0x7fbfffffu;
constexpr uint32_t kNegZero = 0x80000000u;   // accumulator marker of the -0 mode (conv_fwd)

// Key arrays of either width (spc_map_t::key_bits): 64-bit keys, or the 32-bit "Sparse 32"
// storage of Table 1 (valid below 2^32 keys). Indexing reads one key as uint64.
struct Keys {
    const void* p;
    int k32;
    __host__ __device__ Keys() : p(nullptr), k32(0) {}
    __host__ __device__ Keys(const uint64_t* q) : p(q), k32(0) {}
    __host__ __device__ Keys(const void* q, int is32) : p(q), k32(is32) {}
    __device__ __forceinline__ uint64_t operator[](int64_t i) const {
        return k32 ? (uint64_t)__ldg(static_cast<const uint32_t*>(p) + i) : __ldg(static_cast<const uint64_t*>(p) + i);
    }
    // key width known at compile time (hot kernels are instantiated per width)
    template <bool K32>
    __device__ __forceinline__ uint64_t at(int64_t i) const {
        return K32 ? (uint64_t)__ldg(static_cast<const uint32_t*>(p) + i) : __ldg(static_cast<const uint64_t*>(p) + i);
    }
    // low 32 bits of key i (the whole key in 32-bit storage)
    __device__ __forceinline__ uint32_t lo(int64_t i) const {
        return k32 ? __ldg(static_cast<const uint32_t*>(p) + i) : __ldg(static_cast<const uint32_t*>(p) + 2 * i);
    }
    __host__ __device__ explicit operator bool() const { return p != nullptr; }
};
struct KeysOut {
    void* p;
    int k32;
    __host__ __device__ KeysOut() : p(nullptr), k32(0) {}
    __host__ __device__ KeysOut(uint64_t* q) : p(q), k32(0) {}
    __host__ __device__ KeysOut(void* q, int is32) : p(q), k32(is32) {}
    __device__ __forceinline__ void put(int64_t i, uint64_t v) const {
        if (k32) static_cast<uint32_t*>(p)[i] = (uint32_t)v;
        else static_cast<uint64_t*>(p)[i] = v;
    }
    template <bool K32>
    __device__ __forceinline__ void put_t(int64_t i, uint64_t v) const {
        if (K32) static_cast<uint32_t*>(p)[i] = (uint32_t)v;
        else static_cast<uint64_t*>(p)[i] = v;
    }
};

// Geometry of a feature map with its spatial dims padded to rank 4 (leading 1s):
// key = seg*V + ((w*X + x)*Y + y)*Z + z, seg = b*C + c. A "row" is (seg, w, x, y): the Z
// consecutive keys of the last spatial dimension; a "plane" is (w, x): P = w*X + x, so that rank
// <= 3 maps (W = 1) and rank-4 maps share one row / plane layout.
struct Geo {
    int64_t B, C;
    int W, X, Y, Z;
    int64_t V;   // W*X*Y*Z
    int64_t R;   // rows per segment = W*X*Y
};

// Filter geometry padded to rank 4; h = ksize/2 (centre).
struct KGeo {
    int kw, kx, ky, kz;
    int hw, hx, hy, hz;
    int KV;
};

// Filter table meta.x of the backward: the output channel (low 21 bits) and the w-offset
// ow + 512 (bits 21..30); meta.y: pack_off(ox, oy, oz).
__host__ __device__ inline int pack_oc_ow(int oc, int ow) { return oc | ((ow + 512) << 21); }
__device__ __forceinline__ int meta_oc(int m) { return m & 0x1fffff; }
__device__ __forceinline__ int meta_ow(int m) { return ((m >> 21) & 1023) - 512; }

// Packed signed offset o = delta - centre per dim, 10 bits each (|o| < 512).
__host__ __device__ inline int pack_off(int ox, int oy, int oz) {
    return (ox + 512) | ((oy + 512) << 10) | ((oz + 512) << 20);
}
__device__ __forceinline__ int off_x(int p) { return (p & 1023) - 512; }
__device__ __forceinline__ int off_y(int p) { return ((p >> 10) & 1023) - 512; }
__device__ __forceinline__ int off_z(int p) { return ((p >> 20) & 1023) - 512; }

// Order-preserving u32 scores of fp32 values (reading R7: -0 == +0, larger = stronger).
__device__ __forceinline__ uint32_t score_bits(uint32_t bits, int attn) {
    if (attn == SPC_ATTN_MAGNITUDE) return bits & 0x7fffffffu;
    if (bits == 0x80000000u) bits = 0u;                       // -0 -> +0
    return (bits & 0x80000000u) ? ~bits : (bits | 0x80000000u);
}

// Order-preserving u32 of a float for max-pooling; never 0 for non-NaN inputs (0 = empty).
__device__ __forceinline__ uint32_t orderable(float v) {
    uint32_t b = __float_as_uint(v);
    if (b == 0x80000000u) b = 0u;
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float from_orderable(uint32_t o) {
    uint32_t b = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(b);
}

// fast y = L / Z for L < 2^24 (float reciprocal + one correction each way)
__device__ __forceinline__ uint32_t div_small(uint32_t L, uint32_t Z, float invZ) {
    uint32_t q = __float2uint_rz(__uint2float_rz(L) * invZ);
    if (q * Z > L) --q;
    if ((q + 1) * Z <= L) ++q;
    return q;
}

// n / d for 0 <= n < 2^31 by a multiply-high and a shift (d fixed per launch, set on the host):
// m = ceil(2^p / d) with p = 31 + ceil(log2 d), quotient = umulhi(n, m) >> (p - 32); d = 1 is
// m = 0.
struct FastDiv {
    uint32_t d, m, s;
};
inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f{d, 0u, 0u};
    if (d > 1) {
        uint32_t l = 0;
        while ((1ull << l) < d) ++l;   // ceil(log2 d)
        const uint32_t p = 31 + l;
        f.m = (uint32_t)(((1ull << p) + d - 1) / d);
        f.s = p - 32;
    }
    return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
    return f.m ? __umulhi(n, f.m) >> f.s : n;
}

__device__ __forceinline__ int64_t load_n(const int64_t* nnz_dev, int64_t bound) {
    if (!nnz_dev) return bound;
    int64_t n = *nnz_dev;
    return n < bound ? n : bound;
}

// ------------------------------------------------------------- device properties (prof.cu)
// SM count and SM clock (kHz) of the current device, queried once per device (grid sizing and
// the AUTO variant cost model; 148 / 1965000 on B200).
int num_sms();
double sm_clock_hz();

// ------------------------------------------------------------- launch accounting (prof.cu)
void note_launch(int n = 1);
struct PhaseScope {
    PhaseScope(const char* name, cudaStream_t s);
    ~PhaseScope();
    const char* name_;
    cudaStream_t s_;
    cudaEvent_t a_, b_;
};
#define SPC_CAT2(a, b) a##b
#define SPC_CAT(a, b) SPC_CAT2(a, b)
// Brackets the kernel launches of the enclosing scope (one kernel = one note_launch).
#define SPC_PHASE(name, stream, nk) \
    ::spc::note_launch(nk);         \
    ::spc::PhaseScope SPC_CAT(_spc_phase_, __LINE__)(name, stream)

// ------------------------------------------------------------------ launchers (host)
// Row index: row_ptr[r] = first entry with key >= r*Z, r in [0, B*C*R]; workspace
// (B*C*R + 1) uint32 words. Requires nnz < 2^32. With vals / guard: also the forward's value
// guard (*guard = 1 when some stored |x| < 2^-50; *guard must be zeroed before).
cudaError_t launch_row_index(const Geo& g, Keys keys, const int64_t* nnz_dev, int64_t nnz_bound,
                             uint32_t* row_ptr, cudaStream_t s, const float* vals = nullptr, int* guard = nullptr);

// Segment bounds: seg_ptr[s] = first entry with key >= s*V, s in [0, nseg] (nseg + 1 words).
cudaError_t launch_seg_bounds(Keys keys, const int64_t* nnz_dev, int64_t nbound, int64_t nseg, int64_t V,
                              uint32_t* seg_ptr, cudaStream_t s);

// Filter table in ic-major order. meta[j] = {oc, packed offset}; val[j]; off[ic*(c_out+1)+oc]
// = first table entry of (ic, oc) (off[ic*(c_out+1)+c_out] = end); src[j] = original filter
// position of table entry j. scratch: 2*c_in*c_out ints.
cudaError_t launch_filter_table(const KGeo& kg, int c_in, int c_out, const uint64_t* wkeys, const float* wvals,
                                int64_t nw, int2* meta, float* val, int* off, int* src, int* scratch, cudaStream_t s);

// Second filter order for the forward kernel: (ic, dxdy, oc, dz); meta2 = {oc, oz}.
// scratch: 2 * c_in * kx*ky * c_out ints.
cudaError_t launch_filter_table_fwd(const KGeo& kg, int c_in, int c_out, const uint64_t* wkeys, const float* wvals,
                                    int64_t nw, int2* meta2, float* val2, int* off2, int* scratch, cudaStream_t s);

// Forward tile: one x-plane, rows [y0, y0+TY) (full Z), a group of ocg output channels (warp w
// accumulates channel oc0 + w). Tiles of a segment are in key order: ti = x*nty + ty.
struct FwdTile {
    int TY, nty, ocg, n_ocg;
    int ZR;            // accumulator row pitch (floats)
    int cz;            // accumulator column of z = 0 (>= hz, multiple of 4)
    int RA;            // accumulator rows per output channel: TY + 4*hy (margin mode) or TY (pred mode)
    int pred;          // 1: no margin rows, updates leaving the band predicated off
    int PK;            // work items (ic, input plane) = c_in * kx
    int nwg_max;       // stored weights of one output-channel group (upper bound = round records)
    int rec_smem;      // 1: round records copied to shared memory; 0: read through L1
    FastDiv fd_nty, fd_X;   // tile index -> (plane, band), plane -> (w, x)
    FastDiv fd_Z;           // voxel of a band -> (row, z) in the candidate epilogue
    size_t smem;
};
FwdTile plan_fwd_tile(const Geo& gy, const KGeo& kg, int c_out, int c_in, int64_t nw_total, double rho_in);

// Per-segment selection state of the forward (attention) pipeline.
struct FwdSeg {
    uint64_t kstar;      // keep an entry iff composite(score, p) >= kstar
    int64_t need;        // candidates to select
    uint32_t b1;         // threshold digit (11 bits)
    int32_t keep_all;    // 1: keep every support entry
};
// Split resolve (few segments): the bucket / narrowing outcome of a segment, handed from
// stream_resolve_kernel to the multi-CTA collect and the final select.
struct ResolveState {
    uint64_t pre;        // survivors: (K' >> pos) == pre
    uint64_t need;       // survivors to select
    uint32_t B, lo;      // threshold digit, its lowest score
    int32_t pos, sh1;
    int32_t active;      // 1: collect + select pending
    int32_t pad;
};
struct FwdArgs {
    Keys xkeys;
    const int64_t* x_nnz_dev;        // device-side input count (or null: x_nnz)
    int64_t x_nnz;
    const float* xvals;
    const uint32_t* xrow;
    const int2* meta2;
    const float* val2;
    const int* off2;
    int2* rnd;                       // [n_ocg * nwg_max] weight rounds {byte offset, w} (fwd_rounds)
    int* roff;                       // [n_ocg * (ocg * PK + 1)] first round of each (oc, ic, input plane)
    int* guard;                      // set when some |x| or |w| < 2^-50: NaN-marker accumulation
    const float* bias;
    int attn;
    int64_t k;
    float* pre;                      // [nseg * V] pre-attention responses (absent marker off support)
    int64_t nchunk;                  // chunks of 4096 voxels per (b, oc) buffer
    int64_t nseg;                    // (b, oc) segments
    unsigned long long* seg_count;   // [nseg] support size
    uint32_t* hist;                  // [nseg * kSelBins]
    uint32_t* rhist;                 // [nseg * kSelBins] resolve histogram built by several CTAs per
                                     // segment (few segments: batch 1 on large grids), or null
    ResolveState* rstate;            // [nseg] (split resolve)
    uint64_t* rsurv;                 // [nseg * 4096] survivors of the threshold bucket (split resolve)
    uint32_t* rsurv_n;               // [nseg]
    FwdSeg* seg;                     // [nseg]
    uint32_t* tile_def;              // [nseg * nchunk] entries kept outright per chunk
    uint32_t* tile_sel;              // [nseg * nchunk] selected candidates per chunk
    uint64_t* tile_off;              // [nseg * nchunk] output offset of a chunk within its segment
    uint64_t* cand_off;              // [nseg + 1] candidate list offsets
    uint64_t* cand_cnt;              // [nseg] candidates per segment
    unsigned long long* cand_cur;    // [nseg] append cursors
    uint2* cand;                     // candidate list {p, value bits}
    uint2* stg;                      // staged entries with digit >= B1 {p, value bits}, per chunk in key order
    uint64_t* stg_cnt;               // [nseg] staged entries per segment (histogram count of digits >= B1)
    uint64_t* stg_off;               // [nseg + 1] staging offsets
    unsigned long long* stg_cur;     // [nseg] chunk placement cursors
    uint64_t* chunk_stg;             // [nseg * nchunk] first staged entry of each chunk
    uint32_t* chunk_ge;              // [nseg * nchunk] staged entries of each chunk
    uint64_t* seg_off;               // [nseg + 1] output offsets
    KeysOut out_keys;
    float* out_vals;
    int64_t* out_nnz;
    // batch-sliced passes (sparse_conv_fwd_pass): this pass covers samples b0 .. b0 + gy.B - 1;
    // segment s of the pass is global segment b0 * c_out + s; out_append: the pass's outputs go
    // after the *out_nnz entries already written (and *out_nnz grows by them)
    int64_t b0, seg0;
    int out_append;
    int guard_done;   // the value guard ran with the row index (launch_row_index with vals)
    // ---- streamed forward (variant S, launch_conv_fwd_stream): the pre-attention responses
    // never leave the SM. A sampled pass estimates a per-segment score threshold tlow; the main
    // pass appends every support entry with score >= tlow (the candidates, a superset of the k
    // kept ones) to the segment's run for the tile, in key order; an exact selection over the
    // candidates and an ordered write follow. Tile t of a segment = x*nty + ty; its run starts at
    // the tile's first voxel (x*Y + ty*TY)*Z of the segment's candidate region (it holds at most
    // the tile's voxels).
    int ntile;                       // tiles per segment (X * nty)
    int nsamp, sp_period, sp_off;    // sampled tiles per segment: t = j*sp_period + sp_off
    FastDiv fd_ntile, fd_nsamp;      // block index decode of the tile kernels
    uint32_t* tlow;                  // [nseg] candidate score threshold (0: every support entry)
    uint32_t* cmax;                  // [nseg] largest candidate score
    uint32_t* cpos;                  // [nseg * V] candidate spatial index p
    float* cval;                     // [nseg * V] candidate value (bias added)
    uint32_t* tcnt;                  // [nseg * ntile] candidates of each tile run
    int* fail;                       // [nseg] 1: the candidates missed the k-th score (redo pass)
    int* bflag;                      // [B] sample queued for the redo pass
    int* redo_b;                     // [B] queued samples
    int* redo_n;                     // number of queued samples
    int seg_stride;                  // c_out (segment s belongs to sample s / c_out of the pass)
};
// Variant G of the forward accumulate (conv_gemm.cu): tcgen05 TF32 (3xTF32) implicit GEMM over
// filter offsets, writing the same dense pre-attention buffer as the scatter kernel.
struct GemmPlan {
    int ok;            // 1 if the layer fits the variant (c_in <= 32, c_out <= 64)
    int Kp, Np, KV;    // K = c_in padded to 8, N = c_out padded to 16, filter offsets
    int64_t ntile;     // 128-voxel tiles per sample
    int tcols;         // TMEM columns allocated per CTA
    int stages;        // operand stages in shared memory
    size_t stage_bytes, smem;
    // slab form (conv_gemm_slab_kernel): tile 16 rows x 8 z, neighbourhood SX x SY x SZ voxels
    int slab, SX, SY, SZ, NV, nty, ntz, bstages, ball, bgroup, nacc, tcols_slab;
    int kparts, Kh;    // slab K split: the channels in kparts parts of Kh (2 parts: two CTAs per SM)
    size_t slab_bytes, bstage_bytes, slab_smem;
};
struct GemmArgs {
    Keys xkeys;
    const float* xvals;
    const int64_t* x_nnz_dev;
    int64_t x_nnz;
    const uint64_t* wkeys;
    const float* wvals;
    int64_t nw;
    const uint32_t* xrow;   // row index of the input (tiled densify)
    float* xhi;        // [B*V*Kp] dense input, TF32 high part (zero off the support)
    float* xlo;        // [B*V*Kp] low part
    uint32_t* occ;     // [B*V] occupancy mask over ic
    float* bhi;        // [KV*Np*Kp] per-offset B (canonical K-major layout), high part
    float* blo;        // low part
    uint32_t* wmask;   // [KV*Np] stored-weight mask over ic
    int* dinfo;        // [3*KV + 1] offsets with weights, uniform-mask flags, slab offsets
    const float* bias;
    float* pre;
};
GemmPlan plan_gemm(const Geo& gx, const Geo& gy, const KGeo& kg);
cudaError_t launch_conv_gemm(const Geo& gx, const Geo& gy, const KGeo& kg, const GemmPlan& g, const GemmArgs& ga,
                             const FwdArgs& a, cudaStream_t s);

// Streamed forward (variant S, no dense buffer): sampled threshold pass, candidate pass, exact
// selection over the candidates (with a redo pass for segments whose sample missed), ordered
// write. FwdArgs' streamed fields must be carved (a.pre / stg / cand are unused).
cudaError_t launch_conv_fwd_stream(const Geo& gx, const Geo& gy, const KGeo& kg, const FwdTile& t,
                                   const FwdArgs& a, cudaStream_t s);
// sampling plan of the streamed forward (sets a->ntile / nsamp / sp_period / sp_off)
void plan_fwd_sampling(const Geo& gy, const FwdTile& t, int attn, FwdArgs* a);
// per-segment stages of the streamed forward (fwd_stream.cu)
cudaError_t launch_stream_find(const FwdArgs& a, cudaStream_t s);
cudaError_t launch_stream_resolve(const Geo& gy, const FwdTile& t, const FwdArgs& a, int pass, cudaStream_t s);
cudaError_t launch_stream_tail(const Geo& gy, const FwdTile& t, const FwdArgs& a, cudaStream_t s);
// exclusive scan of a per-segment u64 array (one block); total -> *total; add_base: start at
// *total (appending passes of the batch-sliced forward)
cudaError_t launch_seg_scan_u64(const uint64_t* in, uint64_t* out, int64_t n, int64_t* total, int add_base,
                                cudaStream_t s);

// Dense-buffer pipeline (variant G): the accumulate stage writes the dense pre-attention buffer
// that the classify / resolve / write stages read.
cudaError_t launch_conv_fwd_pipeline(const Geo& gx, const Geo& gy, const KGeo& kg, const FwdTile& t,
                                     const FwdArgs& a, cudaStream_t s, const GemmPlan* gp = nullptr,
                                     const GemmArgs* ga = nullptr);

struct BwdTile {
    int TX, TY, ocg, ntx, nty, n_ocg, grid;
    int ocp, ocs;     // passes per item, output channels per pass (ocg = ocp * ocs)
    FastDiv fd_tiles, fd_W, fd_ntx, fd_HWX, fd_HX, fd_TX;   // ntx*nty, W, ntx, HW*HX, HX, TX
    int sY, sX, sW, sOC;   // G slab strides (floats), bank-spread padding
    int threads;      // CTA size (512: one CTA per SM, 256: two)
    int nwg_max;      // upper bound of stored weights in one output-channel group
    size_t smem;
};
BwdTile plan_bwd_tile(const Geo& gx, const KGeo& kg, int c_out, int n_w_max_group);
cudaError_t launch_conv_bwd(const Geo& gx, const Geo& gy, const KGeo& kg, const BwdTile& t,
                            Keys xkeys, const float* xvals, const uint32_t* xrow,
                            Keys ykeys, const float* dy, const uint32_t* yrow,
                            const int2* wmeta, const float* wval, const int* woff, const int* wsrc,
                            float* dx, double* dw_acc, bool want_dx, bool want_dw, cudaStream_t s);
cudaError_t launch_dbias(const Geo& gy, const uint32_t* yrow, const float* dy, double* db_acc, cudaStream_t s);
cudaError_t launch_f64_to_f32(const double* a, float* b, int64_t n, cudaStream_t s);
cudaError_t launch_f64_to_f32_2(const double* a, float* b, int64_t n, const double* a2, float* b2, int64_t n2,
                                cudaStream_t s);

// ---------------------------------------------------------------- selection (attention)
constexpr int kSelBins = 2048;    // 11-bit score digits
// Standalone attention over a COO map (select.cu): segment s = entries row_ptr[s*R] ..
// row_ptr[(s+1)*R]; workspace seg_off [nseg].
struct TkSeg;
// workspace of the streamed top-k (select.cu); tiles = topk_tiles_bound(nnz, nseg)
struct TopkBufs {
    uint64_t* seg_off;      // [nseg + 1] output offset of each segment
    uint32_t* tile_start;   // [nseg + 1] first tile of each segment
    uint32_t* hist;         // [nseg << topk_bits(nnz, nseg)]
    TkSeg* seg;             // [nseg]
    uint32_t* cand_cnt;     // [nseg]
    uint64_t* cand;         // [nnz] candidate composites (segment s at its entry offset)
    uint32_t* tile_seg;     // [tiles] segment of each tile
    uint32_t* tile_def;     // [tiles]
    uint32_t* tile_sel;     // [tiles]
    uint64_t* tile_off;     // [tiles]
};
size_t topk_tiles_bound(int64_t nnz, int64_t nseg);
size_t topk_seg_bytes();
int topk_bits(int64_t nnz, int64_t nseg);   // width of the first score digit (11 or 13)
cudaError_t launch_topk(Keys keys, const float* vals, const uint32_t* seg_lo, int64_t nseg, int64_t nnz_bound,
                        int attn, int64_t k, const TopkBufs& w, KeysOut out_keys, float* out_vals,
                        int64_t* out_src, int64_t* out_nnz, cudaStream_t s);

// --------------------------------------------------------------------- relu / pool / misc
cudaError_t launch_relu(Keys keys, const float* vals, const int64_t* nnz_dev, int64_t nbound,
                        uint32_t* chunk_cnt, uint64_t* chunk_off, uint64_t* scan_tmp,
                        KeysOut out_keys, float* out_vals, int64_t* out_src, int64_t* out_nnz, cudaStream_t s);
struct PoolPlan {
    int sw, sx, sy, sz;
    int PW, PX, PY, PZ;   // pooled dims
    int zchunk;           // pooled z positions per work item
    int nzc;              // z chunks per pooled row
    int64_t items;        // work items: B*C*PX*PY*nzc (row form) or the tiles (tile form)
    int tiled;            // tile form: one CTA per (b, c, pooled plane, band of nyb pooled rows)
    int nyb, nyt;         // pooled rows per tile, tiles per pooled plane
    uint32_t mZ, msy, msz;  // floor((2^32 - 1) / d) for d = Z, sy, sz (division by multiply-high)
    int lZ, lsy, lsz;       // log2 of Z, sy, sz when a power of two (a shift), else -1
};
PoolPlan plan_pool(const Geo& g, int sw, int sx, int sy, int sz);
// Tile form (p.tiled): row_ptr is the band-bound workspace (pool_bound_words), filled here;
// row form: the map's row index (launch_row_index) built by the caller.
size_t pool_bound_words(const Geo& g, const PoolPlan& p);
cudaError_t launch_maxpool(const Geo& g, const PoolPlan& p, Keys keys, const float* vals, const int64_t* nnz_dev,
                           int64_t nbound, const uint32_t* row_ptr, uint32_t* item_cnt, uint64_t* item_off, uint64_t* scan_tmp,
                           KeysOut out_keys, float* out_vals, int64_t* out_arg, int64_t* out_nnz, cudaStream_t s);
cudaError_t launch_scatter_grad(const int64_t* src, const float* dy, int64_t n_out_bound, const int64_t* n_out_dev,
                                float* dx, int64_t n_in, cudaStream_t s);
cudaError_t launch_scatter_grad_sorted(const int64_t* src, const float* dy, int64_t n_out_bound,
                                       const int64_t* n_out_dev, float* dx, int64_t n_in, cudaStream_t s);
cudaError_t launch_check_sorted(const int64_t* src, int64_t n_out_bound, const int64_t* n_out_dev, int64_t n_in,
                                int* flag, cudaStream_t s);

// Device-wide exclusive scan of uint32 counts into uint64 offsets; total -> *total (int64,
// may be NULL). tmp: scan_tmp_words(n) uint64 words.
size_t scan_tmp_words(int64_t n);
cudaError_t launch_scan_u32(const uint32_t* in, uint64_t* out, int64_t n, int64_t* total, uint64_t* tmp,
                            cudaStream_t s);

// ------------------------------------------------------------- training-loop steps (train.cu)
struct DensityReg {
    double lambda, rho_up, o, b1, b2;
};
cudaError_t launch_adagrad(float* w, const float* g, float* acc, int64_t n, const int64_t* y_nnz_dev, double y_cells,
                           const DensityReg& reg, bool has_reg, double lr, double eps, cudaStream_t s);
size_t prune_ws_words(int64_t n);
cudaError_t launch_prune(const uint64_t* keys, const float* w, const float* acc, const uint8_t* warn, int64_t n,
                         double eps, uint64_t* ok, float* ow, float* oacc, uint8_t* owarn, int64_t* out_nnz,
                         uint64_t* ws, cudaStream_t s);

// sparseToDense bridge (index.cu)
cudaError_t launch_to_dense(Keys keys, const float* vals, const int64_t* nnz_dev, int64_t bound,
                            float* dense, int64_t cells, cudaStream_t s);
cudaError_t launch_gather_dense(Keys keys, const int64_t* nnz_dev, int64_t bound, const float* ddense,
                                float* dvals, cudaStream_t s);

struct CodecGeo {
    int nd;
    int64_t B, C;
    int64_t d[SPC_MAX_NDIM];
    uint64_t V, total;   // prod(dims), B*C*V
};
cudaError_t launch_encode_keys(const CodecGeo& g, const int64_t* coords, int64_t n, uint64_t* keys, int* bad,
                               cudaStream_t s);
cudaError_t launch_decode_keys(const CodecGeo& g, const uint64_t* keys, int64_t n, int64_t* coords, int* bad,
                               cudaStream_t s);
cudaError_t launch_keys_narrow(const uint64_t* keys, const int64_t* nnz_dev, int64_t bound, uint32_t* out, cudaStream_t s);
cudaError_t launch_keys_widen(const uint32_t* keys, const int64_t* nnz_dev, int64_t bound, uint64_t* out, cudaStream_t s);
// Validation (SPC_VALIDATE=1): flag = 1 if keys are not strictly increasing or out of range.
cudaError_t launch_validate(Keys keys, const int64_t* nnz_dev, int64_t nbound, uint64_t limit,
                            int* flag, cudaStream_t s);

}  // namespace spc

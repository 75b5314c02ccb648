/*
 * spconv.h — C-ABI of libspconv.so, the B200 (sm_100a) hot path of
 * Hackel et al., arXiv 1801.10585, "Inference, Learning and Attention Mechanisms that
 * Exploit and Preserve Sparsity in Convolutional Networks".
 *
 * Citations: "P:n" = PAPER.md line n (the paper text); readings R1..R13 are in DESIGN.md.
 *
 * ----------------------------------------------------------------------------------------
 * Data format (reading R11)
 *   A sparse feature map is a coordinate list: strictly increasing 64-bit keys and fp32
 *   values in separate device arrays ("indices ... and the corresponding data entries in
 *   separate tensors"; "64 bit keys, and 32 bit depth for feature maps").
 *     key = ((b * channels + c) * V + row_major(p)),   V = prod(dims),
 *   with the first spatial dimension most significant, so keys sort by batch, then channel
 *   ("sorted w.r.t. batches and within each batch w.r.t. channels").
 *   A filter bank is a coordinate list over (oc, ic, delta):
 *     key = ((oc * c_in + ic) * prod(ksize) + row_major(delta)), strictly increasing
 *   ("sorted w.r.t. the output channels and within each channel w.r.t. the input channels").
 *
 * Conventions (all functions)
 *   - Every array argument is a DEVICE pointer; the descriptor structs themselves, stride[]
 *     and k are HOST values. Calls are stream-ordered and asynchronous: they enqueue work on
 *     `stream` and return without synchronising (except SPC_VALIDATE=1, see Errors).
 *   - Ownership: every buffer (inputs, outputs, workspace, nnz words) belongs to the caller and
 *     must stay alive until the enqueued work completes. The library keeps no pointer after
 *     returning and allocates no device memory; it is re-entrant for distinct workspaces.
 *   - Sizes: an input map's exact nnz is *nnz_dev when nnz_dev != NULL (a device int64; `nnz`
 *     is then an upper bound used for grid sizing), else `nnz`. Outputs write their exact
 *     count to *nnz_dev (device) so chained layers never need a host sync.
 *   - Spatial rank 1..4 (SPC_MAX_NDIM; "generic n-dimensional tensors"); odd kernel sizes;
 *     prod(ksize) <= 1024. The tensor-core accumulate variant (SPC_VARIANT_GEMM) is rank <= 3.
 *   - Row length (last dimension Z): the scatter forward keeps one band row of Z + 2hz fp32
 *     columns per output channel on chip (up to ~50 k columns); the backward keeps a gradient
 *     slab of (1 + 2hw)(TX + 2hx)(TY + 2hy)(Z + 2hz) fp32 words (1D up to ~50 k columns, 2D with
 *     ky = 3 ~17 k, 3D with 3x3 ~5.5 k). Longer rows return SPC_ERR_UNSUPPORTED.
 *   - Convolution is cross-correlation with SAME zero padding and stride 1 (readings R1, R2).
 *   - Workspace: query the byte count with the matching *_query function, pass a device
 *     buffer of at least that many bytes (256-byte aligned).
 *
 * Errors
 *   Host-checkable problems (NULL pointers, ndim out of range, even ksize, c_in mismatch,
 *   k < 1 with attention on, capacity or workspace too small) return synchronously with
 *   nothing enqueued. With the environment variable SPC_VALIDATE=1 every input map (and the
 *   filter keys) is also checked on the device (strictly increasing, in range); that check synchronises the
 *   stream and returns SPC_ERR_UNSORTED on failure. Without it, unsorted or duplicate keys
 *   give unspecified values but every write stays within the output capacity. CUDA launch
 *   failures return SPC_ERR_CUDA.
 * ----------------------------------------------------------------------------------------
 */
#ifndef SPCONV_H
#define SPCONV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* cudaStream_t;

#define SPC_MAX_NDIM 4

typedef enum {
    SPC_OK = 0,
    SPC_ERR_INVALID_ARG = 1,
    SPC_ERR_SHAPE = 2,
    SPC_ERR_CAPACITY = 3,
    SPC_ERR_WORKSPACE = 4,
    SPC_ERR_UNSORTED = 5,
    SPC_ERR_UNSUPPORTED = 6,
    SPC_ERR_CUDA = 7
} spc_status_t;

/* Attention variants: (i) raw responses, (ii) absolute values. */
typedef enum {
    SPC_ATTN_NONE = 0,      /* exact convolution, no k-selection                      */
    SPC_ATTN_MAGNITUDE = 1, /* variant (ii): keep the k largest |y|                    */
    SPC_ATTN_RAW = 2        /* variant (i):  keep the k largest y                      */
} spc_attn_t;

/* Input sparse feature map. */
typedef struct {
    int32_t ndim;                  /* spatial rank k of Eq. (1), 1..4                    */
    int64_t batch;                 /* b                                                  */
    int64_t channels;              /* c                                                  */
    int64_t dims[SPC_MAX_NDIM];    /* s_d per spatial dim (first = most significant)     */
    int64_t nnz;                   /* exact count, or upper bound if nnz_dev != NULL     */
    const int64_t* nnz_dev;        /* device: exact count, or NULL                       */
    const uint64_t* keys;          /* device [nnz], strictly increasing                  */
    const float* values;           /* device [nnz]                                       */
    int32_t key_bits;              /* 0 or 64: keys are uint64; 32: `keys` points to uint32
                                      keys ("Sparse 32", Table 1, App. A),
                                      valid when batch*channels*prod(dims) <= 2^32       */
} spc_map_t;

/* Output sparse feature map (shape implied by the operation). */
typedef struct {
    int64_t capacity;              /* entries available in keys/values (and index arrays) */
    uint64_t* keys;                /* device [capacity]                                   */
    float* values;                 /* device [capacity]                                   */
    int64_t* nnz_dev;              /* device: receives the exact output count             */
    int32_t key_bits;              /* 0 or 64: uint64 keys; 32: uint32 keys (as spc_map_t) */
} spc_map_out_t;

/* Sparse filter bank; nnz entries = the unpruned weights (rho_f of Eq. (1)). */
typedef struct {
    int32_t ndim;
    int64_t c_in, c_out;
    int64_t ksize[SPC_MAX_NDIM];   /* odd, s_f per spatial dim                            */
    int64_t nnz;
    const uint64_t* keys;          /* device [nnz], strictly increasing                   */
    const float* values;           /* device [nnz]                                        */
} spc_filter_t;

const char* spc_version(void);
const char* spc_status_string(spc_status_t s);

/* ------------------------------------------------------------------------------------
 * sparse_conv_fwd — Direct Sparse Convolution with Attention, Alg. 1 (§3.1-3.2).
 *   For every (b, oc): accumulate val*fval at uid = id - fid + centre over all stored inputs
 *   and stored weights; the pre-attention set is the structural support S(b,oc) of
 *   those updates (reading R3); bias[oc] is added on S only (R4); if attn !=
 *   NONE and |S| > k, keep the k entries with the largest score (|y| or y), ties by smaller
 *   spatial key (R5-R7); write keys ((b*c_out + oc)*V + p) in key order.
 *   x: input map (channels == w->c_in); w: filter; bias: device [c_out] or NULL (zero);
 *   y: output, capacity >= spc_conv_fwd_query's out_capacity = batch*c_out*min(k, V)
 *   (attention) or batch*c_out*V (none); output shape (batch, c_out, dims).
 *   Guarantees nnz(b, oc) <= k, i.e. output density <= k/V per channel.
 * ------------------------------------------------------------------------------------ */
spc_status_t spc_conv_fwd_query(const spc_map_t* x, const spc_filter_t* w, spc_attn_t attn, int64_t k,
                                int64_t* out_capacity, size_t* workspace_bytes);
spc_status_t sparse_conv_fwd(const spc_map_t* x, const spc_filter_t* w, const float* bias,
                             spc_attn_t attn, int64_t k, spc_map_out_t* y,
                             void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* Accumulate variants of the forward. Both compute the sum of Alg. 1
 * and the same structural support, then share the attention stage.
 *   SCATTER: each stored input times each stored weight, read-modify-write into a shared-memory
 *            slice of the dense buffer -- work proportional to Eq. (1)'s pairs.
 *   GEMM:    output-stationary contraction over (filter offset, c_in) on the tensor cores
 *            (tcgen05 kind::tf32, 3xTF32 split for fp32 accuracy) -- work proportional to the grid;
 *            for layers whose rows are dense (c_in <= 32, c_out <= 64; more workspace: a dense
 *            copy of the input, 8*c_in bytes + 4 per voxel).
 *   AUTO:    the cheaper one by a cost model (sparse_conv_fwd); the Python layer replaces the model
 *            by a measurement per layer.
 * Unsupported explicit choices return SPC_ERR_UNSUPPORTED. spc_conv_fwd_variant() reports which
 * variant a call would run (SPC_VARIANT_SCATTER or SPC_VARIANT_GEMM; 0 on invalid arguments). */
typedef enum { SPC_VARIANT_AUTO = 0, SPC_VARIANT_SCATTER = 1, SPC_VARIANT_GEMM = 2 } spc_variant_t;
spc_status_t spc_conv_fwd_query_ex(const spc_map_t* x, const spc_filter_t* w, spc_attn_t attn, int64_t k,
                                   spc_variant_t variant, int64_t* out_capacity, size_t* workspace_bytes);
spc_status_t sparse_conv_fwd_ex(const spc_map_t* x, const spc_filter_t* w, const float* bias,
                                spc_attn_t attn, int64_t k, spc_variant_t variant, spc_map_out_t* y,
                                void* workspace, size_t workspace_bytes, cudaStream_t stream);
int spc_conv_fwd_variant(const spc_map_t* x, const spc_filter_t* w, spc_attn_t attn, int64_t k,
                         spc_variant_t variant);

/* Batch-sliced forward (memory). The paper keeps ONE temporary dense buffer and
 * reuses it across (b, oc) (Table 1 "Sparse Temp" = r^k * 8 bytes, Appendix A
 * "a temporary buffer, which can be reused in all layers"). sparse_conv_fwd holds the buffer,
 * candidate and staging lists of every (b, oc) at once (fastest: one launch per stage for the
 * whole batch); sparse_conv_fwd_pass sizes them for samples_per_pass samples and runs
 * ceil(batch / samples_per_pass) passes of the scatter pipeline on `stream`, appending each
 * pass's outputs in key order -- the output is identical (bit for bit) to sparse_conv_fwd's
 * scatter variant. samples_per_pass: 1..batch, 0 = batch. Workspace from
 * spc_conv_fwd_query_pass (same samples_per_pass); out_capacity as spc_conv_fwd_query.
 * Errors: as sparse_conv_fwd; SPC_ERR_UNSUPPORTED when the scatter variant does not fit. */
spc_status_t spc_conv_fwd_query_pass(const spc_map_t* x, const spc_filter_t* w, spc_attn_t attn, int64_t k,
                                     int64_t samples_per_pass, int64_t* out_capacity, size_t* workspace_bytes);
spc_status_t sparse_conv_fwd_pass(const spc_map_t* x, const spc_filter_t* w, const float* bias,
                                  spc_attn_t attn, int64_t k, int64_t samples_per_pass, spc_map_out_t* y,
                                  void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* ------------------------------------------------------------------------------------
 * Backward of the convolution, Alg. 2 with the masked rule of Eqs. (3)/(4)
 * (P:121-129): gradients exist only at stored inputs and stored (unpruned) weights.
 *   y: the forward OUTPUT map (its keys are the kept entries; values unused);
 *   dy: device [nnz(y)] gradient aligned with y's keys (attention-dropped outputs carry no
 *   gradient, reading R10);
 *   dx: device [nnz(x)] aligned with x's keys (fixed shape, P:135 (i));
 *   dw: device [w->nnz] aligned with w's keys (pruned weights have no storage and stay 0,
 *   P:135 (iii)); dbias: device [c_out] = sum of dy per output channel, or NULL.
 *   dx accumulates in fp32; dw and dbias accumulate in fp64 and are rounded once.
 * sparse_conv_bwd computes all three in one pass over the (input, weight) pairs as Alg. 2
 * does; the _input / _weight entry points compute one side each.
 * ------------------------------------------------------------------------------------ */
spc_status_t spc_conv_bwd_query(const spc_map_t* x, const spc_filter_t* w, const spc_map_t* y,
                                size_t* workspace_bytes);
spc_status_t sparse_conv_bwd(const spc_map_t* x, const spc_filter_t* w, const spc_map_t* y,
                             const float* dy, float* dx, float* dw, float* dbias,
                             void* workspace, size_t workspace_bytes, cudaStream_t stream);
spc_status_t sparse_conv_bwd_input(const spc_map_t* x, const spc_filter_t* w, const spc_map_t* y,
                                   const float* dy, float* dx,
                                   void* workspace, size_t workspace_bytes, cudaStream_t stream);
spc_status_t sparse_conv_bwd_weight(const spc_map_t* x, const spc_filter_t* w, const spc_map_t* y,
                                    const float* dy, float* dw, float* dbias,
                                    void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* sparse_conv_bwd_f64 -- the data-parallel form of sparse_conv_bwd (SURVEY §8 a11 / e): dx as in
 * sparse_conv_bwd (fp32; NULL to skip), dw64 / dbias64 = the UNROUNDED fp64 accumulators of this
 * call (device [w->nnz] / [c_out] doubles, overwritten; dbias64 may be NULL). Alg. 2 sums
 * bp_filter over the batch: each rank computes the fp64 partial of its sample shard, the
 * partials are summed across ranks (NCCL all-reduce, SUM -- reading R13) and spc_round_f64 rounds
 * the sum once, so the sharded dw equals the single-GPU dw bit for bit whenever the fp64 sums
 * are exact (and to 1 ulp otherwise). Workspace from spc_conv_bwd_query. Errors: as
 * sparse_conv_bwd; SPC_ERR_INVALID_ARG when dw64 is NULL. */
spc_status_t sparse_conv_bwd_f64(const spc_map_t* x, const spc_filter_t* w, const spc_map_t* y,
                                 const float* dy, float* dx, double* dw64, double* dbias64,
                                 void* workspace, size_t workspace_bytes, cudaStream_t stream);
/* spc_round_f64 -- out[i] = (float)in[i], round to nearest even, i < n (device pointers);
 * the single rounding of the reduced fp64 gradients (R12). */
spc_status_t spc_round_f64(const double* in, float* out, int64_t n, cudaStream_t stream);

/* ------------------------------------------------------------------------------------
 * attention_topk — the attention filter as a standalone layer: per (b, c)
 * segment of x keep min(k, n_seg) entries with the largest score (|v| for MAGNITUDE, v for
 * RAW; ties by smaller key, R7); output in key order with x's shape.
 *   src_index: device [capacity] int64 (input position of each kept entry) or NULL.
 *   out capacity >= min(nnz(x), batch*channels*min(k, V)).
 * ------------------------------------------------------------------------------------ */
spc_status_t spc_topk_query(const spc_map_t* x, spc_attn_t attn, int64_t k,
                            int64_t* out_capacity, size_t* workspace_bytes);
spc_status_t attention_topk(const spc_map_t* x, spc_attn_t attn, int64_t k, spc_map_out_t* y,
                            int64_t* src_index, void* workspace, size_t workspace_bytes,
                            cudaStream_t stream);

/* ------------------------------------------------------------------------------------
 * sparse_relu — sparse ReLU ("truncates negative activations"): keep entries
 * with v > 0 (R9), order preserved. src_index: device [capacity] int64 or NULL.
 * out capacity >= nnz(x).
 * ------------------------------------------------------------------------------------ */
spc_status_t spc_relu_query(const spc_map_t* x, int64_t* out_capacity, size_t* workspace_bytes);
spc_status_t sparse_relu(const spc_map_t* x, spc_map_out_t* y, int64_t* src_index,
                         void* workspace, size_t workspace_bytes, cudaStream_t stream);

/* ------------------------------------------------------------------------------------
 * sparse_maxpool — sparse max-pooling, §3.3: entries are assigned to the pooled
 * voxel floor(p / stride) ("dividing ... their index by strides"), and the max is taken per
 * cluster (R8: window = stride, output dims ceil(d / stride), max over stored entries only,
 * empty clusters absent). argmax: device [capacity] int64, the input position of the
 * maximum (ties -> smaller input key), or NULL. stride: HOST [ndim] positive integers.
 * out capacity >= nnz(x). The algorithm is sort-free, unlike the paper's sort.
 * ------------------------------------------------------------------------------------ */
spc_status_t spc_maxpool_query(const spc_map_t* x, const int64_t* stride,
                               int64_t* out_capacity, size_t* workspace_bytes);
spc_status_t sparse_maxpool(const spc_map_t* x, const int64_t* stride, spc_map_out_t* y,
                            int64_t* argmax, void* workspace, size_t workspace_bytes,
                            cudaStream_t stream);

/* ------------------------------------------------------------------------------------
 * sparse_scatter_grad — backward of ReLU / max-pool / attention_topk (Eq. (5)):
 *   dx[0..n_in) = 0, then dx[src_index[t]] = dy[t] for t < n_out. src_index must be
 *   injective (it is for all three layers). n_out = *n_out_dev if non-NULL (bounded by
 *   n_out_bound), else n_out_bound.
 * ------------------------------------------------------------------------------------ */
spc_status_t sparse_scatter_grad(const int64_t* src_index, const float* dy, int64_t n_out_bound,
                                 const int64_t* n_out_dev, float* dx, int64_t n_in,
                                 cudaStream_t stream);

/* sparse_scatter_grad_sorted — the same result when src_index[0..n_out) is strictly increasing
 *   (ReLU and attention_topk emit their sources in key order; max-pool's argmax is not
 *   ordered): every dx element is written once (dy at a source, 0 on the gaps), no separate
 *   zero fill, so the call moves exactly its compulsory bytes. Unsorted or out-of-range input
 *   gives an unspecified dx; under SPC_VALIDATE=1 it returns SPC_ERR_UNSORTED instead
 *   (synchronising). */
spc_status_t sparse_scatter_grad_sorted(const int64_t* src_index, const float* dy, int64_t n_out_bound,
                                        const int64_t* n_out_dev, float* dx, int64_t n_in,
                                        cudaStream_t stream);

/* ------------------------------------------------------------------------------------
 * spc_encode_keys / spc_decode_keys — the key codec of §3 (indices "compressed into
 *   unique 1D keys and only expanded when needed"; Alg. 1 line 1: "decompress filter and
 *   data indices from 1D to kD"): key = (b*channels + c)*prod(dims) + row_major(p), the first
 *   spatial dim most significant (reading R11) -- the keys every op here takes.
 *   coords: device int64 [n][2 + ndim], rows (b, c, p_0 .. p_{ndim-1}); keys: device uint64 [n];
 *   dims: host int64 [ndim]. encode: a row with a coordinate outside [0, extent) gets key
 *   UINT64_MAX and sets *bad_dev = 1; decode: a key >= batch*channels*prod(dims) gets the
 *   coordinates -1 and sets *bad_dev = 1 (bad_dev: device int written only on such an entry, may
 *   be NULL). Host-checkable problems (ndim outside 1..4, non-positive extents, key space above
 *   2^63, null arrays with n > 0, n < 0) return SPC_ERR_INVALID_ARG / SPC_ERR_SHAPE with nothing
 *   enqueued. Asynchronous on `stream`; caller-owned buffers.
 * ------------------------------------------------------------------------------------ */
spc_status_t spc_encode_keys(int32_t ndim, int64_t batch, int64_t channels, const int64_t* dims,
                             const int64_t* coords, int64_t n, uint64_t* keys, int* bad_dev, cudaStream_t stream);
spc_status_t spc_decode_keys(int32_t ndim, int64_t batch, int64_t channels, const int64_t* dims,
                             const uint64_t* keys, int64_t n, int64_t* coords, int* bad_dev, cudaStream_t stream);

/* ------------------------------------------------------------------------------------
 * sparse_to_dense — the sparseToDense() bridge of the OctNet3 stacks (Appendix B, Table 2,
 *   P:332): dense[key] = value for every stored entry, 0 elsewhere. dense: device float
 *   [batch*channels*prod(dims)] in [b][c][dims] order (the key layout makes the key the linear
 *   index, reading R11). sparse_to_dense_bwd: dvalues[i] = ddense[key_i] (the gradient flows only
 *   to stored entries). Errors: null pointers, bad shape -> SPC_ERR_INVALID_ARG/SHAPE.
 * ------------------------------------------------------------------------------------ */
spc_status_t sparse_to_dense(const spc_map_t* x, float* dense, cudaStream_t stream);
spc_status_t sparse_to_dense_bwd(const spc_map_t* x, const float* ddense, float* dvalues, cudaStream_t stream);

/* ------------------------------------------------------------------------------------
 * Memory model (§3, Table 1, §4.1, Appendix A).
 *
 * spc_memory_estimate — the paper's theoretical footprint of one layer's result (host only, no
 *   GPU work): cells = r^ndim,
 *     dense  = cells * batch * channels * 4                          (fp32 dense tensor)
 *     sparse = ceil(rho_up * cells) * batch * channels * (index_bits/8 + 4)   (keys + fp32)
 *     temp   = cells * 8                                  (one reused 64-bit buffer per voxel)
 *   (reading R15). index_bits 32 or 64. SPC_ERR_UNSUPPORTED for 32-bit indices when
 *   cells*batch*channels >= 2^32 (Appendix A: "32 bit indices can only be used for resolutions
 *   r < 256^3 due to buffer overflows"; Table 1 prints "-" there). Outputs in bytes (NULL = skip).
 *
 * sparse_keys_narrow / sparse_keys_widen — the "Sparse 32" storage of Table 1: keys32[i] =
 *   (uint32_t)keys[i] and back, for maps whose key space batch*channels*prod(dims) < 2^32
 *   (else SPC_ERR_UNSUPPORTED). 8 instead of 12 bytes per stored entry between layers; the
 *   layer kernels take 64-bit keys. Device arrays of nnz (bound) entries; the device count
 *   nnz_dev (or nnz) limits the copy. Asynchronous on `stream`.
 * ------------------------------------------------------------------------------------ */
spc_status_t spc_memory_estimate(int32_t ndim, int64_t r, int64_t batch, int64_t channels, double rho_up,
                                 int32_t index_bits, double* dense_bytes, double* sparse_bytes,
                                 double* temp_bytes);
spc_status_t sparse_keys_narrow(const spc_map_t* x, uint32_t* keys32, cudaStream_t stream);
spc_status_t sparse_keys_widen(const uint32_t* keys32, const int64_t* nnz_dev, int64_t nnz, uint64_t* keys,
                               cudaStream_t stream);

/* ------------------------------------------------------------------------------------
 * Spatial sharding of one sample across ranks (beyond the paper, whose dense
 * temporary buffer holds a whole (b, oc) grid on one GPU). The FIRST spatial dimension
 * ("planes", most significant in the key, R11) is cut into contiguous ranges; rank r owns the
 * outputs of planes [a_r, e_r) and needs the inputs of planes [a_r - h, e_r + h), h = ksize[0]/2
 * (Eq. (1): an output depends on inputs within the filter's extent). A shard map is an ordinary
 * map over dims (e_r - a_r, dims[1..]) with the same batch and channels; plane = prod(dims[1..]).
 * 64-bit keys only (SPC_ERR_UNSUPPORTED otherwise). Asynchronous on `stream`; device arrays.
 *
 * spc_slab_gather — for every segment s = b*channels + c (nseg of them), the concatenation over
 *   sources j = 0..nsrc-1 (nsrc <= 4) of source j's entries of segment s with plane in
 *   [lo_j, hi_j) (source coordinates), each re-based to plane + shift_j of an output grid of
 *   `planes_out` planes:  out_key = key + s*(planes_out - planes_j)*plane + shift_j*plane.
 *   The output is sorted when the sources' shifted ranges are disjoint and increasing in j
 *   (halo assembly: left halo, own planes, right halo; owned-plane extraction and shard <->
 *   global re-basing are nsrc = 1). src_index (optional, [capacity]) receives base_j + e for
 *   source entry e, base_j = n_0 + ... + n_{j-1} (the sources' `n` bounds): the position in the
 *   concatenated source index space (halo partial gradients are routed with it). Source j's
 *   count is *nnz_dev when non-NULL, else n. y->capacity >= sum n_j; *y->nnz_dev = exact count.
 *   Workspace from spc_slab_gather_query (3 words per (segment, source)).
 *
 * spc_topk_digit_hist / spc_topk_digit_pick / spc_topk_keep_ge — the attention k-selection of
 *   P:80-84 (§3.2; variants P:104) over a segment split across ranks, as an exact 8-round
 *   radix select on the composite c = (score << 32) | ~(uint32)(p + p_base) of reading R7
 *   (score: |y| for MAGNITUDE, sign-folded y for RAW; p = key mod prod(dims), the shard-local
 *   position; p_base = a_r*plane makes it the global one, so ties break as on one GPU;
 *   p + p_base < 2^32 required). Per-segment device state: prefix[nseg] (uint64, zeroed
 *   before round 1), need[nseg] (int64, = k before round 1; < 0 = settled), hist[nseg*256]
 *   (uint32, zeroed before each round). For shift = 56, 48, ..., 0:
 *     digit_hist: hist[s][d] += #{entries of s with (c >> (shift+8)) == (prefix[s] >> (shift+8))
 *                 and ((c >> shift) & 255) == d}   (all entries when shift = 56)
 *     (the caller sums hist over ranks: one all-reduce per round)
 *     digit_pick: the digit d with above(d) < need[s] <= above(d) + hist[s][d] (above = the
 *                 count of larger digits): prefix[s] |= d << shift, need[s] -= above(d); in
 *                 round 1 a segment with at most need[s] entries in total keeps all of them
 *                 (prefix 0, need -1: "keep all if |S| <= k").
 *   After round shift = 0, prefix[s] is the k-th largest composite of the whole segment (or 0).
 *   spc_topk_keep_ge writes the entries with c >= thr[seg] in key order (src_index optional:
 *   their input positions); y->capacity >= x->nnz; workspace from spc_topk_keep_query.
 *
 * spc_index_add — out[idx[t]] += v[t], t < n (n = *n_dev if non-NULL, bounded by n_bound);
 *   idx must be injective (halo partials of dx added into the owner's dx).
 * ------------------------------------------------------------------------------------ */
typedef struct {
    const uint64_t* keys;          /* device [n], sorted                                     */
    const float* values;           /* device [n]                                             */
    const int64_t* nnz_dev;        /* device exact count, or NULL (then n)                   */
    int64_t n;                     /* count, or upper bound when nnz_dev != NULL             */
    int64_t planes;                /* planes of the source grid                              */
    int64_t lo, hi;                /* kept planes [lo, hi), source coordinates               */
    int64_t shift;                 /* output plane = source plane + shift                    */
} spc_slab_src_t;

spc_status_t spc_slab_gather_query(int64_t nseg, int32_t nsrc, size_t* workspace_bytes);
spc_status_t spc_slab_gather(const spc_slab_src_t* srcs, int32_t nsrc, int64_t nseg, int64_t plane,
                             int64_t planes_out, spc_map_out_t* y, int64_t* src_index, void* workspace,
                             size_t workspace_bytes, cudaStream_t stream);
spc_status_t spc_topk_digit_hist(const spc_map_t* x, spc_attn_t attn, int64_t p_base, const uint64_t* prefix,
                                 const int64_t* need, int32_t shift, uint32_t* hist, cudaStream_t stream);
spc_status_t spc_topk_digit_pick(int64_t nseg, const uint32_t* hist, int32_t shift, uint64_t* prefix,
                                 int64_t* need, cudaStream_t stream);
spc_status_t spc_topk_keep_query(const spc_map_t* x, size_t* workspace_bytes);
spc_status_t spc_topk_keep_ge(const spc_map_t* x, spc_attn_t attn, int64_t p_base, const uint64_t* thr,
                              spc_map_out_t* y, int64_t* src_index, void* workspace, size_t workspace_bytes,
                              cudaStream_t stream);
spc_status_t spc_index_add(const int64_t* idx, const float* v, int64_t n_bound, const int64_t* n_dev,
                           float* out, cudaStream_t stream);

/* ------------------------------------------------------------------------------------
 * Training-loop steps over a sparse filter bank. Elementwise over the STORED
 * weights only: pruned weights are absent and therefore never move or reappear.
 *
 * sparse_adagrad_step — §4 "stochastic gradient descent with the adagrad optimizer" with the
 *   adaptive density regulariser of §3.5: the regulariser sum (w + b)^2 adds
 *   2*lambda*(w + b) to the data gradient, with Eq. (6)
 *     b = o + b1*(rho - rho_up)   if rho > rho_up   ("exceeds available resources")
 *     b = -b2*(rho_up - rho)      otherwise          ("not using available resources")
 *   and rho = *y_nnz_dev / y_cells, the measured density of the layer's output (device word of
 *   the forward, so no host synchronisation). Per parameter, in double precision:
 *     g = grad + 2 lambda (w + b);  a = accum + g^2;  w -= lr g / (sqrt(a) + eps);  accum = a.
 *   params/grad/accum: device float [n] (params and accum updated in place); reg: host struct or
 *   NULL (no regulariser; then y_nnz_dev may be NULL). Errors: n < 0, null arrays with n > 0,
 *   reg given without y_nnz_dev or y_cells <= 0 -> SPC_ERR_INVALID_ARG.
 *
 * sparse_filter_prune — one-warning-shot pruning at an epoch end, §3.6: a stored
 *   weight with |w| < eps whose warning flag is set is removed; |w| < eps otherwise sets the flag
 *   (the warning shot); |w| >= eps clears it. keys/values/accum/warn (device, [n]; accum may be
 *   NULL) are compacted together in key order into the out_* arrays (capacity n); the new count
 *   goes to *out_nnz_dev. The paper's eps is 0.01 (Appendix B). Workspace: spc_prune_query.
 * ------------------------------------------------------------------------------------ */
typedef struct {
    double lambda;   /* regularisation scale (the paper sweeps 0 .. 0.3, §4.3)            */
    double rho_up;   /* upper density bound implied by the k-selection                    */
    double o, b1, b2;/* Eq. (6) control parameters (>= 0; the paper uses 0.1 each)        */
} spc_density_reg_t;
spc_status_t sparse_adagrad_step(float* params, const float* grad, float* accum, int64_t n,
                                 const int64_t* y_nnz_dev, double y_cells, const spc_density_reg_t* reg,
                                 double lr, double eps, cudaStream_t stream);
spc_status_t spc_prune_query(int64_t n, size_t* workspace_bytes);
spc_status_t sparse_filter_prune(const uint64_t* keys, const float* values, const float* accum,
                                 const uint8_t* warn, int64_t n, double eps, uint64_t* out_keys,
                                 float* out_values, float* out_accum, uint8_t* out_warn,
                                 int64_t* out_nnz_dev, void* workspace, size_t workspace_bytes,
                                 cudaStream_t stream);

/* ------------------------------------------------------------------------------------
 * Instrumentation (measurement only; not part of the method).
 *   spc_kernel_launches: monotonically increasing count of kernels this library launched
 *   (process-wide).
 *   spc_profile_enable(1): every kernel phase is bracketed by CUDA events recorded on the
 *   call's stream; spc_profile_read synchronises those events and returns, per phase name,
 *   the accumulated milliseconds and the number of launches (names are written NUL-separated
 *   into `names`; returns the number of phases). spc_profile_reset clears the totals.
 * ------------------------------------------------------------------------------------ */
int64_t spc_kernel_launches(void);
spc_status_t spc_profile_enable(int on);
spc_status_t spc_profile_reset(void);
int spc_profile_read(char* names, size_t names_len, double* ms, int64_t* counts, int max_phases);

#ifdef __cplusplus
}
#endif

#endif /* SPCONV_H */

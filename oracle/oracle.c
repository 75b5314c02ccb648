/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the hot path of
 * Hackel et al., arXiv 1801.10585 ("Inference, Learning and Attention Mechanisms that
 * Exploit and Preserve Sparsity in CNNs"). It exists to prove the CUDA path right.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it. It shares no code, header or constant with paper_1801_10585_b200/ and the
 * product path never calls it.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n. Readings R1..R13 are listed in
 * DESIGN.md ("Readings of the paper").
 *
 * Arithmetic: all accumulation in fp64 (double); results rounded to fp32 once, because
 * the paper stores "32 bit depth for feature maps". Single-threaded, scalar loops,
 * no blocking, fusion or reordering beyond the paper's own loop nests.
 *
 * Layout (R11): feature-map key = ((b*C + c)*V + row_major(p)), first spatial dim most
 * significant; filter key = ((oc*c_in + ic)*prod(ksize) + row_major(delta)).
 *
 * Return codes: 0 ok, -1 invalid argument, -2 keys unsorted/duplicate, -3 key out of range,
 * -4 output capacity too small, -5 out of memory.
 *
 * Pinning: every function here is pinned by tests/test_oracle_pins.py against brute force
 * (dense fp64 convolution / autograd in torch on CPU, full sorts in Python), the SPEC worked
 * examples (tests/golden/) and the paper's invariants. No function is "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define ORA_MAXDIM 4

/* ---------------------------------------------------------------- key codec */
/* P:43 "indices of the form {batch, index_x, index_y, ..., channel} are compressed into
 * unique 1D keys and only expanded when needed"; P:45 sort order batch -> channel. */

static int64_t volume_of(int ndim, const int64_t* dims) {
    int64_t v = 1;
    for (int d = 0; d < ndim; ++d) v *= dims[d];
    return v;
}

/* decode key -> (b, c, p[0..ndim)) ; returns 0 or -3 when out of range */
static int decode_key(uint64_t key, int ndim, const int64_t* dims, int64_t batch, int64_t channels,
                      int64_t* b, int64_t* c, int64_t* p) {
    int64_t V = volume_of(ndim, dims);
    uint64_t total = (uint64_t)batch * (uint64_t)channels * (uint64_t)V;
    if (key >= total) return -3;
    uint64_t spatial = key % (uint64_t)V;
    uint64_t seg = key / (uint64_t)V;
    *c = (int64_t)(seg % (uint64_t)channels);
    *b = (int64_t)(seg / (uint64_t)channels);
    for (int d = ndim - 1; d >= 0; --d) {
        p[d] = (int64_t)(spatial % (uint64_t)dims[d]);
        spatial /= (uint64_t)dims[d];
    }
    return 0;
}

static uint64_t encode_key(int ndim, const int64_t* dims, int64_t channels,
                           int64_t b, int64_t c, const int64_t* p) {
    uint64_t lin = 0;
    for (int d = 0; d < ndim; ++d) lin = lin * (uint64_t)dims[d] + (uint64_t)p[d];
    return ((uint64_t)b * (uint64_t)channels + (uint64_t)c) * (uint64_t)volume_of(ndim, dims) + lin;
}

int ora_decode_key(uint64_t key, int ndim, const int64_t* dims, int64_t batch, int64_t channels,
                   int64_t* out /* [2+ndim]: b, c, p... */) {
    if (ndim < 1 || ndim > ORA_MAXDIM) return -1;
    return decode_key(key, ndim, dims, batch, channels, &out[0], &out[1], &out[2]);
}

uint64_t ora_encode_key(int ndim, const int64_t* dims, int64_t channels, const int64_t* idx /* b,c,p */) {
    return encode_key(ndim, dims, channels, idx[0], idx[1], &idx[2]);
}

static int check_sorted(int64_t n, const uint64_t* keys) {
    for (int64_t i = 1; i < n; ++i)
        if (keys[i] <= keys[i - 1]) return -2;
    return 0;
}

/* ---------------------------------------------------------- get_update_id */
/* Alg. 1 step "compute uid with get_update_id(id, fid)". Reading R1: cross-correlation,
 * uid = id - fid + centre per spatial dim; reading R2: SAME zero padding, stride 1, a uid
 * outside the grid does not exist. Returns 1 if uid is inside the grid. */
static int get_update_id(int ndim, const int64_t* dims, const int64_t* ksize,
                         const int64_t* id, const int64_t* fid, int64_t* uid) {
    for (int d = 0; d < ndim; ++d) {
        int64_t u = id[d] - fid[d] + ksize[d] / 2;
        if (u < 0 || u >= dims[d]) return 0;
        uid[d] = u;
    }
    return 1;
}

int ora_get_update_id(int ndim, const int64_t* dims, const int64_t* ksize,
                      const int64_t* id, const int64_t* fid, int64_t* uid) {
    return get_update_id(ndim, dims, ksize, id, fid, uid);
}

static int64_t lin_of(int ndim, const int64_t* dims, const int64_t* p) {
    int64_t l = 0;
    for (int d = 0; d < ndim; ++d) l = l * dims[d] + p[d];
    return l;
}

/* segment offsets of a sorted key array: off[s] = first entry with key >= s*span, s in [0, nseg] */
static void segment_offsets(int64_t n, const uint64_t* keys, int64_t nseg, uint64_t span, int64_t* off) {
    int64_t i = 0;
    for (int64_t s = 0; s <= nseg; ++s) {
        uint64_t lo = (uint64_t)s * span;
        while (i < n && keys[i] < lo) ++i;
        off[s] = i;
    }
}

/* -------------------------------------------------------- k-selection (attention) */
/* keep the k strongest responses per output channel; variant (i) raw values,
 * variant (ii) absolute values. Reading R7: total order (score desc, key asc). */
typedef struct { float score; int64_t pos; float value; double abs; int64_t src; } ora_cand;

static int cmp_score_desc_pos_asc(const void* a, const void* b) {
    const ora_cand* x = (const ora_cand*)a;
    const ora_cand* y = (const ora_cand*)b;
    if (x->score > y->score) return -1;
    if (x->score < y->score) return 1;
    return (x->pos < y->pos) ? -1 : (x->pos > y->pos ? 1 : 0);
}

static int cmp_pos_asc(const void* a, const void* b) {
    const ora_cand* x = (const ora_cand*)a;
    const ora_cand* y = (const ora_cand*)b;
    return (x->pos < y->pos) ? -1 : (x->pos > y->pos ? 1 : 0);
}

static float score_of(float v, int attn) {
    /* attn 1 = MAGNITUDE (variant ii), 2 = RAW (variant i). -0 and +0 compare equal as floats. */
    return attn == 1 ? fabsf(v) : v;
}

/* select the first min(k, n) candidates under (score desc, pos asc), then re-sort by pos.
 * Returns the number kept. A full sort: slow and obviously correct. */
static int64_t select_k(ora_cand* cand, int64_t n, int attn, int64_t k) {
    if (attn == 0 || n <= k) return n;
    for (int64_t i = 0; i < n; ++i) cand[i].score = score_of(cand[i].value, attn);
    qsort(cand, (size_t)n, sizeof(ora_cand), cmp_score_desc_pos_asc);
    qsort(cand, (size_t)k, sizeof(ora_cand), cmp_pos_asc);
    return k;
}

/* ------------------------------------------------- Algorithm 1: forward + attention */
/*
 * Direct Sparse Convolution with Attention, Alg. 1:
 *   decompress filter and data indices from 1D to kD
 *   for b, for oc:
 *     initialize dense buffer with 0
 *     for ic, for {id,val} in data(b,ic), for {fid,fval} in filter(oc,ic)
 *       uid = get_update_id(id, fid); buffer[uid] += val*fval
 *     get non-zero entries from buffer  [R3: structural]
 *     add bias to non-zero entries  [R4]
 *     select k largest responses  [R5-R7]
 *     compress ids from kD to 1D, write as sparse output
 *
 * attn: 0 none (exact convolution), 1 magnitude, 2 raw. k: entries kept per (b, oc).
 * Output: y keys/values sorted; y_abs (optional) = sum of |val*fval| + |bias| per output, the
 * scale of the tolerance rule. macs (optional) = number of in-bounds
 * (input, weight) pairs = Eq. (1) first term.
 */
int ora_conv_fwd(int ndim, const int64_t* dims, int64_t batch, int64_t c_in, int64_t c_out,
                 const int64_t* ksize,
                 int64_t nx, const uint64_t* xk, const float* xv,
                 int64_t nw, const uint64_t* wk, const float* wv,
                 const float* bias, int attn, int64_t k,
                 int64_t cap, uint64_t* yk, float* yv, double* yabs, int64_t* ny_out,
                 int64_t* macs_out) {
    if (ndim < 1 || ndim > ORA_MAXDIM || batch < 0 || c_in < 1 || c_out < 1) return -1;
    for (int d = 0; d < ndim; ++d) if (dims[d] < 1 || ksize[d] < 1 || ksize[d] % 2 == 0) return -1;
    if (attn != 0 && k < 1) return -1;
    if (check_sorted(nx, xk) || check_sorted(nw, wk)) return -2;

    const int64_t V = volume_of(ndim, dims);
    const int64_t KV = volume_of(ndim, ksize);
    /* step 1: decompress data and filter indices */
    int64_t* xp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nx > 0 ? nx : 1) * ndim);
    int64_t* wp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nw > 0 ? nw : 1) * ndim);
    int64_t* xoff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(batch * c_in + 1));
    int64_t* woff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(c_out * c_in + 1));
    double* A = (double*)malloc(sizeof(double) * (size_t)V);
    double* Aabs = (double*)malloc(sizeof(double) * (size_t)V);
    char* R = (char*)malloc((size_t)V);
    ora_cand* cand = (ora_cand*)malloc(sizeof(ora_cand) * (size_t)V);
    int rc = 0;
    if (!xp || !wp || !xoff || !woff || !A || !Aabs || !R || !cand) { rc = -5; goto done; }
    for (int64_t i = 0; i < nx; ++i) {
        int64_t b, c;
        if (decode_key(xk[i], ndim, dims, batch, c_in, &b, &c, &xp[i * ndim])) { rc = -3; goto done; }
    }
    for (int64_t j = 0; j < nw; ++j) {
        int64_t oc, ic;
        if (decode_key(wk[j], ndim, ksize, c_out, c_in, &oc, &ic, &wp[j * ndim])) { rc = -3; goto done; }
    }
    segment_offsets(nx, xk, batch * c_in, (uint64_t)V, xoff);
    segment_offsets(nw, wk, c_out * c_in, (uint64_t)KV, woff);

    int64_t ny = 0, macs = 0;
    int64_t uid[ORA_MAXDIM];
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t oc = 0; oc < c_out; ++oc) {
            /* initialize dense buffer with 0 */
            memset(A, 0, sizeof(double) * (size_t)V);
            memset(Aabs, 0, sizeof(double) * (size_t)V);
            memset(R, 0, (size_t)V);
            for (int64_t ic = 0; ic < c_in; ++ic) {
                for (int64_t i = xoff[b * c_in + ic]; i < xoff[b * c_in + ic + 1]; ++i) {
                    for (int64_t j = woff[oc * c_in + ic]; j < woff[oc * c_in + ic + 1]; ++j) {
                        if (!get_update_id(ndim, dims, ksize, &xp[i * ndim], &wp[j * ndim], uid)) continue;
                        int64_t u = lin_of(ndim, dims, uid);
                        double prod = (double)xv[i] * (double)wv[j];
                        A[u] += prod;               /* "add val*fval to buffer at uid" */
                        Aabs[u] += fabs(prod);
                        R[u] = 1;
                        ++macs;
                    }
                }
            }
            /* get non-zero entries (reading R3) + add bias (reading R4) */
            int64_t n = 0;
            double bb = bias ? (double)bias[oc] : 0.0;
            for (int64_t u = 0; u < V; ++u) {
                if (!R[u]) continue;
                cand[n].pos = u;
                cand[n].value = (float)(A[u] + bb);
                cand[n].abs = Aabs[u] + fabs(bb);
                cand[n].src = -1;
                ++n;
            }
            /* select k largest responses */
            int64_t kept = select_k(cand, n, attn, k);
            if (ny + kept > cap) { rc = -4; goto done; }
            /* compress ids from kD to 1D and write */
            for (int64_t t = 0; t < kept; ++t) {
                yk[ny] = (uint64_t)(b * c_out + oc) * (uint64_t)V + (uint64_t)cand[t].pos;
                yv[ny] = cand[t].value;
                if (yabs) yabs[ny] = cand[t].abs;
                ++ny;
            }
        }
    }
    *ny_out = ny;
    if (macs_out) *macs_out = macs;
done:
    free(xp); free(wp); free(xoff); free(woff); free(A); free(Aabs); free(R); free(cand);
    return rc;
}

/* ------------------------------------------------- Algorithm 2: backpropagation */
/*
 * Backpropagation for the convolutional layer, Alg. 2, with the masked rule of
 * Eqs. (3)/(4): gradients exist only for stored inputs and stored weights.
 *   bp_data = 0 (shape of input values); bp_filter = 0 (shape of filter weights)
 *   for b, for oc:
 *     initialize dense buffer with gradients(b, oc)
 *     for ic, {id,val} in data(b,ic), {fid,fval} in filter(oc,ic):
 *       uid = get_update_id(id, fid); g = buffer[uid]
 *       bp_data[id] += g*fval ; bp_filter[fid] += g*val
 * Reading R10: "gradient q" is g = dL/dy at the kept outputs (y keys), 0 elsewhere.
 * dbias[oc] = sum of dy over the kept outputs of channel oc (bias is added on the support only).
 * dx_abs / dw_abs (optional): sums of |terms| for the tolerance rule.
 */
/* dw64 / db64 (optional): the fp64 sums before the final rounding -- the data-parallel tests
 * add these per-shard partials (Alg. 2 sums bp_filter over b; reading R13) and round once. */
int ora_conv_bwd64(int ndim, const int64_t* dims, int64_t batch, int64_t c_in, int64_t c_out,
                   const int64_t* ksize,
                   int64_t nx, const uint64_t* xk, const float* xv,
                   int64_t nw, const uint64_t* wk, const float* wv,
                   int64_t ny, const uint64_t* yk, const float* dy,
                   float* dx, float* dw, float* dbias,
                   double* dx_abs, double* dw_abs, int64_t* kept_pairs_out, double* dw64, double* db64) {
    if (ndim < 1 || ndim > ORA_MAXDIM || batch < 0 || c_in < 1 || c_out < 1) return -1;
    for (int d = 0; d < ndim; ++d) if (dims[d] < 1 || ksize[d] < 1 || ksize[d] % 2 == 0) return -1;
    if (check_sorted(nx, xk) || check_sorted(nw, wk) || check_sorted(ny, yk)) return -2;
    const int64_t V = volume_of(ndim, dims);
    const int64_t KV = volume_of(ndim, ksize);
    int64_t* xp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nx > 0 ? nx : 1) * ndim);
    int64_t* wp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nw > 0 ? nw : 1) * ndim);
    int64_t* xoff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(batch * c_in + 1));
    int64_t* woff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(c_out * c_in + 1));
    int64_t* yoff = (int64_t*)malloc(sizeof(int64_t) * (size_t)(batch * c_out + 1));
    double* G = (double*)malloc(sizeof(double) * (size_t)V);
    char* K = (char*)malloc((size_t)V);
    int64_t kept_pairs = 0;
    double* bpd = (double*)calloc((size_t)(nx > 0 ? nx : 1), sizeof(double));
    double* bpf = (double*)calloc((size_t)(nw > 0 ? nw : 1), sizeof(double));
    double* bpd_abs = (double*)calloc((size_t)(nx > 0 ? nx : 1), sizeof(double));
    double* bpf_abs = (double*)calloc((size_t)(nw > 0 ? nw : 1), sizeof(double));
    int rc = 0;
    if (!xp || !wp || !xoff || !woff || !yoff || !G || !K || !bpd || !bpf || !bpd_abs || !bpf_abs) { rc = -5; goto done; }
    for (int64_t i = 0; i < nx; ++i) {
        int64_t b, c;
        if (decode_key(xk[i], ndim, dims, batch, c_in, &b, &c, &xp[i * ndim])) { rc = -3; goto done; }
    }
    for (int64_t j = 0; j < nw; ++j) {
        int64_t oc, ic;
        if (decode_key(wk[j], ndim, ksize, c_out, c_in, &oc, &ic, &wp[j * ndim])) { rc = -3; goto done; }
    }
    for (int64_t t = 0; t < ny; ++t)
        if (yk[t] >= (uint64_t)(batch * c_out) * (uint64_t)V) { rc = -3; goto done; }
    segment_offsets(nx, xk, batch * c_in, (uint64_t)V, xoff);
    segment_offsets(nw, wk, c_out * c_in, (uint64_t)KV, woff);
    segment_offsets(ny, yk, batch * c_out, (uint64_t)V, yoff);

    int64_t uid[ORA_MAXDIM];
    for (int64_t oc = 0; oc < c_out; ++oc) {
        double db = 0.0;
        for (int64_t b = 0; b < batch; ++b)
            for (int64_t t = yoff[b * c_out + oc]; t < yoff[b * c_out + oc + 1]; ++t) db += (double)dy[t];
        if (dbias) dbias[oc] = (float)db;
        if (db64) db64[oc] = db;
    }
    for (int64_t b = 0; b < batch; ++b) {
        for (int64_t oc = 0; oc < c_out; ++oc) {
            /* initialize dense buffer with gradients(b, oc) */
            memset(G, 0, sizeof(double) * (size_t)V);
            memset(K, 0, (size_t)V);
            for (int64_t t = yoff[b * c_out + oc]; t < yoff[b * c_out + oc + 1]; ++t) {
                G[yk[t] % (uint64_t)V] = (double)dy[t];
                K[yk[t] % (uint64_t)V] = 1;   /* kept output (for the MAC count only) */
            }
            for (int64_t ic = 0; ic < c_in; ++ic) {
                for (int64_t i = xoff[b * c_in + ic]; i < xoff[b * c_in + ic + 1]; ++i) {
                    for (int64_t j = woff[oc * c_in + ic]; j < woff[oc * c_in + ic + 1]; ++j) {
                        if (!get_update_id(ndim, dims, ksize, &xp[i * ndim], &wp[j * ndim], uid)) continue;
                        const int64_t u = lin_of(ndim, dims, uid);
                        double g = G[u];                             /* gradient at uid */
                        kept_pairs += K[u];
                        bpd[i] += g * (double)wv[j];                 /* bp_data[id] += g*fval */
                        bpf[j] += g * (double)xv[i];                 /* bp_filter[fid] += g*val */
                        bpd_abs[i] += fabs(g * (double)wv[j]);
                        bpf_abs[j] += fabs(g * (double)xv[i]);
                    }
                }
            }
        }
    }
    for (int64_t i = 0; i < nx; ++i) { dx[i] = (float)bpd[i]; if (dx_abs) dx_abs[i] = bpd_abs[i]; }
    for (int64_t j = 0; j < nw; ++j) {
        dw[j] = (float)bpf[j];
        if (dw_abs) dw_abs[j] = bpf_abs[j];
        if (dw64) dw64[j] = bpf[j];
    }
    if (kept_pairs_out) *kept_pairs_out = kept_pairs;
done:
    free(xp); free(wp); free(xoff); free(woff); free(yoff); free(G); free(K);
    free(bpd); free(bpf); free(bpd_abs); free(bpf_abs);
    return rc;
}

int ora_conv_bwd(int ndim, const int64_t* dims, int64_t batch, int64_t c_in, int64_t c_out,
                 const int64_t* ksize,
                 int64_t nx, const uint64_t* xk, const float* xv,
                 int64_t nw, const uint64_t* wk, const float* wv,
                 int64_t ny, const uint64_t* yk, const float* dy,
                 float* dx, float* dw, float* dbias,
                 double* dx_abs, double* dw_abs, int64_t* kept_pairs_out) {
    return ora_conv_bwd64(ndim, dims, batch, c_in, c_out, ksize, nx, xk, xv, nw, wk, wv, ny, yk, dy, dx, dw, dbias,
                          dx_abs, dw_abs, kept_pairs_out, NULL, NULL);
}

/* ------------------------------------------------- attention as a standalone layer */
/* P:102-104 k-selection per output channel, applied to a sparse map: per (b, c) segment keep
 * min(k, n_seg) entries by (score desc, key asc); output in key order; src[t] = input index. */
int ora_topk(int ndim, const int64_t* dims, int64_t batch, int64_t channels,
             int64_t nx, const uint64_t* xk, const float* xv, int attn, int64_t k,
             int64_t cap, uint64_t* yk, float* yv, int64_t* src, int64_t* ny_out) {
    if (ndim < 1 || ndim > ORA_MAXDIM || (attn != 1 && attn != 2) || k < 1) return -1;
    if (check_sorted(nx, xk)) return -2;
    const int64_t V = volume_of(ndim, dims);
    if (nx > 0 && xk[nx - 1] >= (uint64_t)(batch * channels) * (uint64_t)V) return -3;
    int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(batch * channels + 1));
    ora_cand* cand = (ora_cand*)malloc(sizeof(ora_cand) * (size_t)(nx > 0 ? nx : 1));
    int rc = 0;
    if (!off || !cand) { rc = -5; goto done; }
    segment_offsets(nx, xk, batch * channels, (uint64_t)V, off);
    int64_t ny = 0;
    for (int64_t s = 0; s < batch * channels; ++s) {
        int64_t n = 0;
        for (int64_t i = off[s]; i < off[s + 1]; ++i) {
            cand[n].pos = (int64_t)xk[i];
            cand[n].value = xv[i];
            cand[n].src = i;
            ++n;
        }
        int64_t kept = select_k(cand, n, attn, k);
        if (ny + kept > cap) { rc = -4; goto done; }
        for (int64_t t = 0; t < kept; ++t) {
            yk[ny] = (uint64_t)cand[t].pos;
            yv[ny] = cand[t].value;
            if (src) src[ny] = cand[t].src;
            ++ny;
        }
    }
    *ny_out = ny;
done:
    free(off); free(cand);
    return rc;
}

/* ------------------------------------------------------------------ sparse ReLU */
/* P:175 "The ReLU, by definition, truncates negative activations to zero"; reading R9: keep
 * v > 0 strictly, order preserved; src[t] = input index. */
int ora_relu(int64_t nx, const uint64_t* xk, const float* xv,
             uint64_t* yk, float* yv, int64_t* src, int64_t* ny_out) {
    int64_t ny = 0;
    for (int64_t i = 0; i < nx; ++i) {
        if (xv[i] > 0.0f) {
            yk[ny] = xk[i];
            yv[ny] = xv[i];
            if (src) src[ny] = i;
            ++ny;
        }
    }
    *ny_out = ny;
    return 0;
}

/* ------------------------------------------------------------- sparse max-pooling */
/*
 * §3.3: "First, features are assigned to an output (hyper-) voxel, by dividing the data
 * channels of their index by strides. Second, the data is sorted w.r.t. voxels, so that all
 * responses within the same voxel are clustered together. Third, the pooling operator is
 * applied separately to each cluster." Reading R8: window = stride, output dims ceil(d/s),
 * max over stored members only, empty cluster -> absent, argmax tie -> smaller input key.
 */
typedef struct { uint64_t pkey; float value; int64_t idx; } ora_pool_item;

static int cmp_pool(const void* a, const void* b) {
    const ora_pool_item* x = (const ora_pool_item*)a;
    const ora_pool_item* y = (const ora_pool_item*)b;
    if (x->pkey != y->pkey) return x->pkey < y->pkey ? -1 : 1;
    if (x->value > y->value) return -1;   /* larger value first */
    if (x->value < y->value) return 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);   /* then smaller input key */
}

int ora_maxpool(int ndim, const int64_t* dims, int64_t batch, int64_t channels, const int64_t* stride,
                int64_t nx, const uint64_t* xk, const float* xv,
                int64_t cap, uint64_t* yk, float* yv, int64_t* argmax, int64_t* ny_out) {
    if (ndim < 1 || ndim > ORA_MAXDIM) return -1;
    for (int d = 0; d < ndim; ++d) if (stride[d] < 1) return -1;
    if (check_sorted(nx, xk)) return -2;
    int64_t odims[ORA_MAXDIM];
    for (int d = 0; d < ndim; ++d) odims[d] = (dims[d] + stride[d] - 1) / stride[d];
    ora_pool_item* it = (ora_pool_item*)malloc(sizeof(ora_pool_item) * (size_t)(nx > 0 ? nx : 1));
    if (!it) return -5;
    int64_t p[ORA_MAXDIM], q[ORA_MAXDIM];
    for (int64_t i = 0; i < nx; ++i) {
        int64_t b, c;
        if (decode_key(xk[i], ndim, dims, batch, channels, &b, &c, p)) { free(it); return -3; }
        for (int d = 0; d < ndim; ++d) q[d] = p[d] / stride[d];   /* divide index by strides */
        it[i].pkey = encode_key(ndim, odims, channels, b, c, q);
        it[i].value = xv[i];
        it[i].idx = i;
    }
    qsort(it, (size_t)nx, sizeof(ora_pool_item), cmp_pool);        /* sort w.r.t. voxels */
    int64_t ny = 0;
    for (int64_t i = 0; i < nx; ++i) {                                /* max per cluster */
        if (i > 0 && it[i].pkey == it[i - 1].pkey) continue;
        if (ny >= cap) { free(it); return -4; }
        yk[ny] = it[i].pkey;
        yv[ny] = it[i].value;
        if (argmax) argmax[ny] = it[i].idx;
        ++ny;
    }
    *ny_out = ny;
    free(it);
    return 0;
}

/* ------------------------------------------- gradient routing for ReLU / pool / top-k */
/* Eq. (5): the gradient passes only where the forward layer kept an entry; pooling
 * routes it to the argmax witness. dx[src[t]] += dy[t], every other dx is 0. */
int ora_scatter_grad(int64_t ny, const int64_t* src, const float* dy, int64_t nx, float* dx) {
    for (int64_t i = 0; i < nx; ++i) dx[i] = 0.0f;
    for (int64_t t = 0; t < ny; ++t) {
        if (src[t] < 0 || src[t] >= nx) return -3;
        dx[src[t]] += dy[t];
    }
    return 0;
}

/* ----------------------------------------------------------- training-loop steps
 * Adaptive density regularisation, §3.5, Eq. (6): the regulariser becomes
 * sum (w + b)^2 with b = o + b1*(rho - rho_up) when rho > rho_up ("exceeds available
 * resources"), and b = -b2*(rho_up - rho) when rho <= rho_up ("not using available resources"). */
double ora_density_bias(double rho, double rho_up, double o, double b1, double b2) {
    if (rho > rho_up) return o + b1 * (rho - rho_up);
    return -b2 * (rho_up - rho);
}

/* One optimiser step over the stored weights (§4: "stochastic gradient descent with the adagrad
 * optimizer"), with the regulariser's gradient lambda * d/dw (w + b)^2 = 2 lambda (w + b) added to
 * the data gradient (§3.5). Per weight, in double precision:
 *   g   = dw + 2 lambda (w + b)
 *   a   = acc + g^2                 (accumulator += grad^2)
 *   w' = w - lr g / (sqrt(a) + eps)
 * then w' and a are stored as fp32. Pruned weights are not stored, so they never move. */
int ora_adagrad_step(int64_t n, float* w, const float* dw, float* acc, double b, double lambda, double lr,
                     double eps) {
    if (n < 0) return -1;
    for (int64_t i = 0; i < n; ++i) {
        double g = (double)dw[i] + 2.0 * lambda * ((double)w[i] + b);
        double a = (double)acc[i] + g * g;
        double wn = (double)w[i] - lr * g / (sqrt(a) + eps);
        acc[i] = (float)a;
        w[i] = (float)wn;
    }
    return 0;
}

/* One-warning-shot pruning at the end of an epoch, §3.6: a stored weight with
 * |w| < eps that was already flagged at the previous epoch end is pruned -- removed from the
 * filter ("zero" = not stored), so it never reappears; |w| < eps without the flag sets
 * the flag (the warning shot); |w| >= eps clears it. Keys, values, accumulators and flags are
 * compacted together in key order. Returns the new count (>= 0) or -1. */
int64_t ora_prune(int64_t n, const uint64_t* keys, const float* w, const float* acc, const uint8_t* warn,
                  double eps, uint64_t* okeys, float* ow, float* oacc, uint8_t* owarn) {
    if (n < 0) return -1;
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i) {
        int small = fabs((double)w[i]) < eps;
        if (small && warn[i]) continue;           /* second consecutive low observation: prune */
        okeys[m] = keys[i];
        ow[m] = w[i];
        oacc[m] = acc[i];
        owarn[m] = (uint8_t)(small ? 1 : 0);       /* warning shot set, or cleared */
        ++m;
    }
    return m;
}

/* sparseToDense() bridge, Appendix B Table 2: dense[b][c][p] = value of the stored entry
 * with key (b, c, p), 0 elsewhere. The dense array is written through decode_key (the key codec of
 * P:43), cell by cell. */
int ora_to_dense(int ndim, const int64_t* dims, int64_t batch, int64_t channels, int64_t n, const uint64_t* keys,
                 const float* vals, float* dense) {
    int64_t V = volume_of(ndim, dims);
    memset(dense, 0, sizeof(float) * (size_t)(batch * channels * V));
    for (int64_t i = 0; i < n; ++i) {
        int64_t b, c, p[ORA_MAXDIM];
        if (decode_key(keys[i], ndim, dims, batch, channels, &b, &c, p) != 0) return -3;
        dense[(b * channels + c) * V + lin_of(ndim, dims, p)] = vals[i];
    }
    return 0;
}

/* ----------------------------------------------------------- memory model
 * Table 1 and Appendix A / Fig. 7: theoretical memory of a layer's
 * result for resolution r (spatial rank k), minibatch b, c output channels, upper bound rho_up.
 *   dense  : one fp32 per grid cell             r^k * b * c * 4      ("Dense convolutions
 *            require only a single output tensor")
 *   sparse : indices and data of the <= rho_up * r^k entries per channel,
 *            ceil(rho_up * r^k) * b * c * (index_bits / 8 + 4)         ("tensors for indices and
 *            data"; 64- or 32-bit indices and "32 bit floating point" data)
 *   temp   : the temporary buffer "which can be reused in all layers", one 64-bit entry
 *            per grid cell, r^k * 8 (reading R15: fits every "Sparse Temp" entry of Table 1)
 * Returns -1 for 32-bit indices when r^k * b * c >= 2^32 ("32 bit indices can only be used for
 * resolutions r < 256^3 due to buffer overflows"; Table 1 prints "-" at 256^3). */
int ora_memory_estimate(int k, int64_t r, int64_t b, int64_t c, double rho_up, int index_bits, double* out3) {
    double cells = 1.0;
    for (int d = 0; d < k; ++d) cells *= (double)r;
    if (index_bits == 32 && cells * (double)b * (double)c >= 4294967296.0) return -1;
    out3[0] = cells * (double)b * (double)c * 4.0;
    out3[1] = ceil(rho_up * cells) * (double)b * (double)c * (double)(index_bits / 8 + 4);
    out3[2] = cells * 8.0;
    return 0;
}

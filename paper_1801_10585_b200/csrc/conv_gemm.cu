// Variant G of the forward accumulate (north star (b)): the same sum as Alg. 1
// (P:60-67), y[b, oc, p] = sum_{delta, ic} x[b, ic, p + delta - c] * w[oc, ic, delta] (reading R1),
// computed output-stationary on the 5th-generation tensor cores for layers whose rows are dense
// enough that a contraction over (delta, ic) is genuine (C3/C5-like channel widths, high density).
//
// Per CTA: one tile of 128 consecutive output voxels of one sample (UMMA M = 128, one TMEM lane
// per voxel) and all output channels (UMMA N = c_out padded to 16). For every filter offset delta
// with a stored weight, the 128 rows of A = x[b, :, p + delta - c] (K = c_in padded to 8) are
// gathered with cp.async from a dense, zero-padded copy of the input into shared memory in the
// canonical K-major layout, B = W_delta is copied likewise, and one elected thread issues
// tcgen05.mma.kind::tf32 into the TMEM accumulator; the gathers of the next offsets overlap the
// MMAs of delta (up to 4 shared-memory stages; full/empty mbarriers, released by tcgen05.commit). fp32 accuracy from TF32 units:
// every operand is split a = hi + lo (hi = a with the low 13 mantissa bits cleared, exact) and
// D += A_hi B_hi + A_hi B_lo + A_lo B_hi (3xTF32; the dropped lo*lo term is < 2^-22 relative).
//
// The epilogue reads the accumulator with tcgen05.ld, applies the structural support of reading
// R3 (a voxel is present for oc iff some stored input meets some stored weight of oc: an OR over
// delta of the input-occupancy masks AND the weight masks), adds the bias on the support
// and writes the same dense pre-attention buffer as the scatter variant (absent marker off the
// support), so the attention pipeline that follows is shared. Support and values therefore match
// variant S exactly in coordinates and within fp32 rounding in value.
#include "spc_internal.cuh"
#include "block_scan.cuh"

#include <algorithm>
#include <cstdlib>

namespace spc {

constexpr int kGM = 128;        // output voxels per tile = UMMA M = TMEM lanes
constexpr int kGThreads = 128;  // thread t gathers A row t and owns TMEM lane t in the epilogue
constexpr int kGMaxStages = 4;  // operand stages in flight (gathers run kGMaxStages - 1 offsets ahead)
constexpr int kSlabTY = 16;     // slab form: M tile = 16 rows x 8 z (a core-matrix group = 8 z of one row)
constexpr int kSlabTZ = 8;
constexpr int kSlabMaxStages = 8;

GemmPlan plan_gemm(const Geo& gx, const Geo& gy, const KGeo& kg) {
    GemmPlan g{};
    const int c_in = (int)gx.C, c_out = (int)gy.C;
    if (c_in < 1 || c_in > 32 || c_out < 1 || c_out > 64) return g;   // masks are u32 over ic; N <= 64
    if (gx.B * gx.C >= (1ll << 32)) return g;                          // 32-bit segment ids in densify
    if (gx.W != 1 || kg.kw != 1) return g;                               // rank <= 3 only (variant S covers rank 4)
    g.Kp = (c_in + 7) & ~7;
    g.Np = (c_out + 15) & ~15;
    g.KV = kg.KV;
    g.ntile = (gy.V + kGM - 1) / kGM;
    g.stage_bytes = (size_t)2 * kGM * g.Kp * 4 + (size_t)2 * g.Np * g.Kp * 4;
    const size_t extra = (size_t)g.KV * g.Np * 4 + (size_t)(3 * g.KV + 1) * 4 + 2 * 8 * std::max(8, g.KV) + 64 + 16;
    int want = 2;   // two stages keep two CTAs (8 warps of gatherers) per SM for the 32-channel layers
    if (const char* e = getenv("SPC_GEMM_STAGES")) want = std::max(2, std::min(kGMaxStages, atoi(e)));
    g.stages = (int)std::min<size_t>((size_t)want, (200 * 1024 - extra) / g.stage_bytes);
    g.smem = g.stages * g.stage_bytes + extra;
    g.tcols = 32;                                        // D = [A.B_hi | A_hi.B_lo]: 2*Np columns
    while (g.tcols < 2 * g.Np) g.tcols *= 2;
    g.ok = g.stages >= 2;
    // slab form: M tile = 16 rows (y) x 8 z of one x-plane; the tile's input neighbourhood is
    // staged once and every A_delta is a strided window of it (no per-offset re-gather)
    g.SX = 1 + 2 * kg.hx;
    g.SY = kSlabTY + 2 * kg.hy;
    g.SZ = kSlabTZ + 2 * kg.hz;
    g.NV = g.SX * g.SY * g.SZ;
    g.nty = (gy.Y + kSlabTY - 1) / kSlabTY;
    g.ntz = (gy.Z + kSlabTZ - 1) / kSlabTZ;
    // K split: the slab holds Kp/2 channels at a time when that lets two CTAs share an SM (the
    // fill of one tile then overlaps the MMAs of the other); else the whole K in one part
    auto slab_plan = [&](int parts, size_t budget) {
        g.kparts = parts;
        g.Kh = g.Kp / parts;
        g.slab_bytes = (size_t)2 * g.NV * g.Kh * 4 + (size_t)g.NV * 4;
        g.bstage_bytes = (size_t)2 * g.Np * g.Kh * 4;
        const size_t room = budget > g.slab_bytes + extra ? budget - g.slab_bytes - extra : 0;
        // every B_delta resident (small filter banks, one part): one load, then all MMAs back to
        // back; otherwise two stages of `bgroup` offsets each (one handshake per group)
        g.ball = parts == 1 && (size_t)g.KV * g.bstage_bytes <= std::min<size_t>(room, 96 * 1024) ? 1 : 0;
        g.bgroup = (int)std::max<size_t>(1, std::min<size_t>(8, room / (2 * g.bstage_bytes)));
        g.bstages = g.ball ? g.KV : 2;
        g.slab_smem = g.slab_bytes + (g.ball ? (size_t)g.KV : (size_t)2 * g.bgroup) * g.bstage_bytes + extra;
        return g.slab_smem <= budget && room >= 2 * g.bstage_bytes;
    };
    const bool split_ok = g.Kp % 16 == 0 && !(getenv("SPC_GEMM_KSPLIT") && getenv("SPC_GEMM_KSPLIT")[0] == '0');
    // 32+ input channels: four K parts of Kp/4 in 56 KB (four CTAs per SM, two TMEM accumulators
    // each: the fills of three tiles overlap the MMAs of the fourth; C5 at 50 %: 2.83 -> 2.61 ms)
    int parts_env = getenv("SPC_GEMM_PARTS") ? atoi(getenv("SPC_GEMM_PARTS")) : (g.Kp % 32 == 0 ? 4 : 0);
    if (parts_env > 0 && g.Kp % (8 * parts_env) == 0 &&
        slab_plan(parts_env, (size_t)(parts_env >= 4 ? 56 : parts_env >= 3 ? 75 : 112) * 1024)) {
        // (planned)
    } else if (!(split_ok && slab_plan(2, 112 * 1024) && slab_plan(1, 200 * 1024) && g.slab_smem > 112 * 1024 &&
                 slab_plan(2, 112 * 1024))) {
        slab_plan(1, 200 * 1024);
    }
    // several TMEM accumulators, offsets dealt round-robin: consecutive MMAs do not depend on
    // each other's result (summed in the epilogue)
    g.nacc = std::max(1, std::min(g.kparts >= 4 ? 2 : 4, 256 / (2 * g.Np)));   // (TMEM shared by 4 CTAs)
    if (const char* e = getenv("SPC_GEMM_NACC")) g.nacc = std::max(1, std::min(g.nacc, atoi(e)));
    g.tcols_slab = 32;
    while (g.tcols_slab < g.nacc * 2 * g.Np) g.tcols_slab *= 2;
    g.slab = (g.slab_smem <= 200 * 1024 && g.NV * 16 < (1 << 18) && g.SZ * 16 < (1 << 18)) ? 1 : 0;
    if (const char* e = getenv("SPC_GEMM_SLAB")) g.slab = g.slab && e[0] != '0';
    return g;
}

// Dense zero-padded copy of the input, split into TF32 hi/lo halves, plus per-voxel occupancy
// masks over ic (a stored 0.0 is occupied: structural support, reading R3).
__global__ void gemm_densify_kernel(Geo gx, int Kp, Keys keys, const float* __restrict__ vals,
                                    const int64_t* nnz_dev, int64_t bound, float* __restrict__ xhi,
                                    float* __restrict__ xlo, uint32_t* __restrict__ occ) {
    const int64_t n = load_n(nnz_dev, bound);
    const double invV = 1.0 / (double)gx.V;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = keys[e];
        // key / V through a double reciprocal (exact after one correction each way; keys < 2^53)
        uint64_t seg = (uint64_t)((double)key * invV);
        if (seg * (uint64_t)gx.V > key) --seg;
        if ((seg + 1) * (uint64_t)gx.V <= key) ++seg;
        const uint64_t p = key - seg * (uint64_t)gx.V;
        const uint32_t s32 = (uint32_t)seg, C32 = (uint32_t)gx.C;   // b*C + ic < 2^32 (checked by the API)
        const uint64_t b = s32 / C32, ic = s32 - (uint32_t)b * C32;
        const float v = vals[e];
        const float hi = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
        const size_t o = (size_t)(b * (uint64_t)gx.V + p) * (size_t)Kp + (size_t)ic;
        xhi[o] = hi;
        xlo[o] = v - hi;
        atomicOr(&occ[b * (uint64_t)gx.V + p], 1u << ic);
    }
}

// Tiled form: one CTA per (b, x, band of ny rows) builds the band's dense [voxel][Kp] block in
// shared memory -- channel c's entries of the band are one contiguous run of the row index -- and
// writes it (and the occupancy masks) with coalesced stores, zeros included (no memset, no
// scattered 4-byte stores). Channel slots are XOR-swizzled by voxel (Kp a power of two) so the
// scatter of one channel's entries hits distinct banks.
__device__ __forceinline__ int dz_slot(int v, int c, int Kp) {
    return (Kp & (Kp - 1)) == 0 ? v * Kp + (c ^ (v & (Kp - 1))) : v * Kp + c;
}

__global__ void __launch_bounds__(256) gemm_densify_tile_kernel(Geo gx, int Kp, int ny, Keys keys,
                                                                 const float* __restrict__ vals,
                                                                 const uint32_t* __restrict__ xrow,
                                                                 float* __restrict__ xhi, float* __restrict__ xlo,
                                                                 uint32_t* __restrict__ occ) {
    extern __shared__ __align__(16) float dsm[];
    const int nyt = (gx.Y + ny - 1) / ny;
    int64_t t = blockIdx.x;
    const int yt = (int)(t % nyt); t /= nyt;
    const int x = (int)(t % gx.X);
    const int64_t b = t / gx.X;
    const int y0 = yt * ny, nyr = min(ny, gx.Y - y0);
    const int Z = gx.Z, TV = nyr * Z, TE = TV * Kp;
    float* shi = dsm;
    float* slo = dsm + (size_t)ny * Z * Kp;
    uint32_t* socc = reinterpret_cast<uint32_t*>(slo + (size_t)ny * Z * Kp);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < TE; i += 256) {
        shi[i] = 0.0f;
        slo[i] = 0.0f;
    }
    for (int v = tid; v < TV; v += 256) socc[v] = 0u;
    __syncthreads();
    for (int c = warp; c < (int)gx.C; c += 8) {
        const int64_t r0 = ((b * gx.C + c) * gx.X + x) * (int64_t)gx.Y + y0;
        const uint32_t e0 = xrow[r0], e1 = xrow[r0 + nyr];
        const uint64_t kb = (uint64_t)r0 * (uint64_t)Z;
        for (uint32_t e = e0 + lane; e < e1; e += 32) {
            const int v = (int)(keys[e] - kb);
            const float val = vals[e];
            const float hi = __uint_as_float(__float_as_uint(val) & 0xffffe000u);
            const int o = dz_slot(v, c, Kp);
            shi[o] = hi;
            slo[o] = val - hi;
            atomicOr(&socc[v], 1u << c);
        }
    }
    __syncthreads();
    const size_t vb = (size_t)b * gx.V + ((size_t)x * gx.Y + y0) * Z;
    for (int i = tid; i < TE; i += 256) {
        const int v = i / Kp, c = i - v * Kp;
        const int o = dz_slot(v, c, Kp);
        xhi[vb * Kp + i] = shi[o];
        xlo[vb * Kp + i] = slo[o];
    }
    for (int v = tid; v < TV; v += 256) occ[vb + v] = socc[v];
}

// element offset of (row, k) in the canonical K-major, no-swizzle UMMA layout of an R-row operand:
// K steps of 8 (32 B per row), 8-row core-matrix groups of 256 B, two 16-byte K halves 128 B apart
__host__ __device__ inline int canon(int row, int k, int R) {
    return (k >> 3) * R * 8 + (row >> 3) * 64 + ((k & 7) >> 2) * 32 + (row & 7) * 4 + (k & 3);
}

// Filter -> per-offset B_delta = [W_hi ; W_lo] (canonical layout, N = 2*c_out rows, K = ic) and
// weight masks over ic. One MMA with the whole operand gives A.W_hi and A.W_lo side by side.
__global__ void gemm_wprep_kernel(KGeo kg, int c_in, int Kp, int Np, const uint64_t* __restrict__ wk,
                                  const float* __restrict__ wv, int64_t nw, float* __restrict__ bhi,
                                  uint32_t* __restrict__ wmask) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nw; j += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = wk[j];
        const int d = (int)(key % (uint64_t)kg.KV);
        const uint64_t r = key / (uint64_t)kg.KV;
        const int ic = (int)(r % (uint64_t)c_in), oc = (int)(r / (uint64_t)c_in);
        const float v = wv[j];
        const float hi = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
        // one N = 2*Np operand per offset: rows [0, Np) the high parts, rows [Np, 2Np) the low parts
        const size_t base = (size_t)d * 2 * Np * Kp;
        bhi[base + canon(oc, ic, 2 * Np)] = hi;
        bhi[base + canon(Np + oc, ic, 2 * Np)] = v - hi;
        atomicOr(&wmask[d * Np + oc], 1u << ic);
    }
}

// Offsets with at least one stored weight (the others contribute nothing) and whether every
// output channel shares the offset's ic mask: dinfo = [nd, dlist[KV], uniform[KV], slab offset[KV]].
__global__ void gemm_dinfo_kernel(KGeo kg, int c_out, int Np, int SY, int SZ, const uint32_t* __restrict__ wmask,
                                  int* __restrict__ dinfo) {
    const int KV = kg.KV;
    if (threadIdx.x == 0) {
        int nd = 0;
        for (int d = 0; d < KV; ++d) {
            uint32_t any = 0, uni = 1;
            for (int oc = 0; oc < c_out; ++oc) {
                any |= wmask[d * Np + oc];
                uni &= (uint32_t)(wmask[d * Np + oc] == wmask[d * Np]);
            }
            if (any) dinfo[1 + nd++] = d;
            dinfo[1 + KV + d] = (int)uni;
            const int dz = d % kg.kz, dy = (d / kg.kz) % kg.ky, dx = d / (kg.kz * kg.ky);
            dinfo[1 + 2 * KV + d] = (dx * SY + dy) * SZ + dz;
        }
        dinfo[0] = nd;
    }
}

// ------------------------------------------------------------------ tcgen05 / mbarrier helpers
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t saddr, uint32_t lbo = 128, uint32_t sbo = 256) {
    // start address >> 4 | LBO (stride between the two 16-byte K halves) >> 4 << 16 | SBO (stride
    // between 8-row core-matrix groups) >> 4 << 32 | version 1 (sm_100) << 46 | SWIZZLE_NONE (0) << 61
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
// Issued by a whole converged warp; elect.sync picks the lane that issues. (Issuing from one
// thread of a divergent warp costs ~150 cycles per MMA -- tools/micro/mma_rate.cu -- against
// 40 cycles for m128n32k8 and 128 for m128n256k8 from a converged warp.)
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
        :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint32_t mbar) {
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" :: "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT%=;\n\t}\n"
        :: "r"(mbar), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t mbar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(mbar) : "memory");
}
// cp.async.wait_group with a runtime bound (the immediate must be a constant)
__device__ __forceinline__ void cp_async_wait_upto(int n) {
    switch (n) {
        case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
        case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
        case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
        case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
        case 4: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
        case 5: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
        default: asm volatile("cp.async.wait_group 6;" ::: "memory"); break;
    }
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void cp4(uint32_t dst, const void* src, bool ok) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" :: "r"(dst), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" :: "r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__global__ void __launch_bounds__(kGThreads) conv_gemm_kernel(Geo gx, Geo gy, KGeo kg, GemmPlan g, GemmArgs a) {
    extern __shared__ __align__(1024) unsigned char gsm[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const int64_t b = blockIdx.x / g.ntile;
    const int64_t p0 = (blockIdx.x - b * g.ntile) * (int64_t)kGM;
    const int Kp = g.Kp, Np = g.Np, KV = g.KV;
    const int c_out = (int)gy.C;
    const size_t A_B = (size_t)kGM * Kp * 4, B_B = (size_t)Np * Kp * 4;
    const int S = g.stages;
    uint32_t* wmask = reinterpret_cast<uint32_t*>(gsm + S * g.stage_bytes);
    int* dlist = reinterpret_cast<int*>(wmask + KV * Np);
    // mbarriers: full[S] (all gatherers arrived) then empty[S] (MMAs of the stage retired)
    uint64_t* mbar = reinterpret_cast<uint64_t*>(gsm + ((S * g.stage_bytes + (size_t)KV * Np * 4 + (size_t)KV * 8 + 7) & ~(size_t)7));
    uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 2 * kGMaxStages);
    __shared__ int s_nd;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(gsm);
    const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(mbar);

    for (int i = tid; i < KV * Np; i += kGThreads) wmask[i] = a.wmask[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"((uint32_t)__cvta_generic_to_shared(tslot)), "r"((uint32_t)g.tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(mb0 + 8u * i, kGThreads);            // full[i]
            mbar_init(mb0 + 8u * (S + i), 1);              // empty[i]
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {   // offsets with at least one stored weight (the others contribute nothing)
        int nd = 0;
        for (int d = 0; d < KV; ++d) {
            uint32_t any = 0, uni = 1;
            for (int oc = 0; oc < c_out; ++oc) {
                any |= wmask[d * Np + oc];
                uni &= (uint32_t)(wmask[d * Np + oc] == wmask[d * Np]);
            }
            if (any) dlist[nd++] = d;
            dlist[KV + d] = (int)uni;   // same ic mask for every oc at this offset
        }
        s_nd = nd;
    }
    const uint32_t tmem = *tslot;

    // this thread's output voxel and its coordinates
    const int64_t p = p0 + tid;
    const bool pin = p < gy.V;
    const int pz = (int)(p % gy.Z), py = (int)((p / gy.Z) % gy.Y), px = (int)(p / ((int64_t)gy.Z * gy.Y));
    __syncthreads();
    const int nd = s_nd;

    auto load_stage = [&](int st, int d) {
        const uint32_t base = sbase + (uint32_t)(st * g.stage_bytes);
        const int dz = d % kg.kz, dy = (d / kg.kz) % kg.ky, dx = d / (kg.kz * kg.ky);
        const int qx = px + dx - kg.hx, qy = py + dy - kg.hy, qz = pz + dz - kg.hz;
        const bool ok = pin && qx >= 0 && qx < gx.X && qy >= 0 && qy < gx.Y && qz >= 0 && qz < gx.Z;
        const size_t q = ok ? ((size_t)b * gx.V + ((size_t)qx * gx.Y + qy) * gx.Z + qz) * Kp : 0;
        const uint32_t rowoff = (uint32_t)((tid >> 3) * 256 + (tid & 7) * 16);
        for (int c = 0; c < Kp / 4; ++c) {   // 16-byte chunks of the row: K step c/2, half c%2
            const uint32_t off = (uint32_t)((c >> 1) * kGM * 32 + (c & 1) * 128) + rowoff;
            cp16(base + off, a.xhi + q + 4 * c, ok);
            cp16(base + (uint32_t)A_B + off, a.xlo + q + 4 * c, ok);
        }
        const float* bh = a.bhi + (size_t)d * 2 * Np * Kp;
        for (int c = tid; c < 2 * Np * Kp / 4; c += kGThreads)
            cp16(base + (uint32_t)(2 * A_B) + 16u * c, bh + 4 * c, true);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(Np >> 3) << 17) | ((uint32_t)(kGM >> 4) << 24);
    const uint32_t idesc2 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)((2 * Np) >> 3) << 17) | ((uint32_t)(kGM >> 4) << 24);

    // Pipeline over the offsets: every thread gathers its A rows (and a share of B) for offset
    // it + S - 1 while the tensor cores work on offset it. full[st] completes when all 128
    // gatherers' cp.async groups for the stage have landed (each waits for its own group, makes
    // it visible to the async proxy, then arrives); empty[st] completes when tcgen05.commit
    // retires the stage's MMAs, after which the stage may be overwritten.
    if (nd > 0) {
        for (int j = 0; j < S - 1; ++j) {
            if (j < nd) load_stage(j, dlist[j]);
            else asm volatile("cp.async.commit_group;" ::: "memory");
        }
        for (int it = 0; it < nd; ++it) {
            const int st = it % S;
            // this thread's group for offset it has landed (younger groups may stay in flight)
            if (S >= 4) asm volatile("cp.async.wait_group 2;" ::: "memory");
            else if (S == 3) asm volatile("cp.async.wait_group 1;" ::: "memory");
            else asm volatile("cp.async.wait_group 0;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_arrive(mb0 + 8u * st);
            if (warp == 0) {   // converged warp: MMAs issued through elect.sync
                mbar_wait(mb0 + 8u * st, (uint32_t)((it / S) & 1));
                tc_fence_after();
                const uint32_t base = sbase + (uint32_t)(st * g.stage_bytes);
                const uint32_t Ah = base, Al = base + (uint32_t)A_B, Bc = base + (uint32_t)(2 * A_B);
                for (int ks = 0; ks < Kp / 8; ++ks) {   // A_hi.[W_hi|W_lo] -> D[:, 0:2Np), A_lo.W_hi -> D[:, 0:Np)
                    const uint64_t db = umma_sdesc(Bc + (uint32_t)(ks * 2 * Np * 32));
                    umma_tf32(tmem, umma_sdesc(Ah + (uint32_t)(ks * kGM * 32)), db, idesc2, (it | ks) != 0);
                    umma_tf32(tmem, umma_sdesc(Al + (uint32_t)(ks * kGM * 32)), db, idesc, 1u);
                }
                umma_commit(mb0 + 8u * (S + st));
            }
            // gather offset it + S - 1 into the slot of offset it - 1 once its MMAs retired
            const int nx = it + S - 1;
            if (nx < nd) {
                if (it >= 1) mbar_wait(mb0 + 8u * (S + (it - 1) % S), (uint32_t)(((it - 1) / S) & 1));
                load_stage(nx % S, dlist[nx]);
            } else {
                asm volatile("cp.async.commit_group;" ::: "memory");
            }
        }
        mbar_wait(mb0 + 8u * (S + (nd - 1) % S), (uint32_t)(((nd - 1) / S) & 1));
        tc_fence_after();
    }

    // ---- epilogue: structural support, bias, dense pre-attention buffer
    // supm bit oc <=> some stored input at p + delta - c meets a stored weight (oc, ic, delta):
    // offsets whose weight masks agree for every oc (dense or uniformly pruned filters) need one
    // test for all channels
    uint64_t supm = 0;
    const uint64_t allm = c_out >= 64 ? ~0ull : ((1ull << c_out) - 1ull);
    if (pin)
        for (int d = 0; d < KV; ++d) {
            const int dz = d % kg.kz, dy = (d / kg.kz) % kg.ky, dx = d / (kg.kz * kg.ky);
            const int qx = px + dx - kg.hx, qy = py + dy - kg.hy, qz = pz + dz - kg.hz;
            if (qx < 0 || qx >= gx.X || qy < 0 || qy >= gx.Y || qz < 0 || qz >= gx.Z) continue;
            const uint32_t nb = a.occ[(size_t)b * gx.V + ((size_t)qx * gx.Y + qy) * gx.Z + qz];
            if (!nb) continue;
            const uint32_t m0 = wmask[d * Np];
            if (dlist[KV + d]) {
                if (nb & m0) supm = allm;
            } else {
                for (int oc = 0; oc < c_out; ++oc)
                    if (nb & wmask[d * Np + oc]) supm |= 1ull << oc;
            }
            if (supm == allm) break;
        }
    for (int c0 = 0; c0 < Np; c0 += 16) {
        float v[16];
        if (nd > 0) {
            float u[16];
            tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
            tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(Np + c0), u);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += u[i];
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = 0.0f;
        }
        if (!pin) continue;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int oc = c0 + i;
            if (oc >= c_out) break;
            const bool sup = (supm >> oc) & 1ull;
            const float bv = a.bias ? __ldg(&a.bias[oc]) : 0.0f;
            a.pre[((size_t)b * c_out + oc) * gy.V + p] = sup ? v[i] + bv : __uint_as_float(kAbsent);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"((uint32_t)g.tcols));
}

// Slab form of variant G. CTA = (b, x, 16 rows from y0, 8 z from z0) = 128 output voxels; M row m
// <-> (y0 + m/8, z0 + m%8), so an 8-row core-matrix group is 8 consecutive z of one row. The
// input neighbourhood (x-hx..x+hx, y0-hy..y0+15+hy, z0-hz..z0+7+hz) is staged ONCE per tile in
// shared memory as [K step][K half][voxel][16 B] (hi and lo copies, plus occupancy masks), and
// A_delta for offset (dx, dy, dz) is the window starting at slab voxel (dx, dy, dz): row group
// stride SBO = SZ*16 B, K-half stride LBO = NV*16 B -- a plain UMMA descriptor, no copy. Only
// B_delta streams per offset (double-buffered, full/empty mbarriers as in the gather form).
__global__ void __launch_bounds__(kGThreads) conv_gemm_slab_kernel(Geo gx, Geo gy, KGeo kg, GemmPlan g, GemmArgs a) {
    extern __shared__ __align__(1024) unsigned char gsm[];
    const int tid = threadIdx.x, warp = tid >> 5;
    const int Kp = g.Kp, Kh = g.Kh, Np = g.Np, KV = g.KV, NV = g.NV, SY = g.SY, SZ = g.SZ;
    const int c_out = (int)gy.C;
    int64_t t = blockIdx.x;
    const int tz = (int)(t % g.ntz); t /= g.ntz;
    const int ty = (int)(t % g.nty); t /= g.nty;
    const int x = (int)(t % gy.X);
    const int64_t b = t / gy.X;
    const int y0 = ty * kSlabTY, z0 = tz * kSlabTZ;
    const int S = g.bstages;
    // shared layout: slab hi | slab lo | occ | B stages | wmask | dlist | mbarriers | tmem slot
    // (the slab holds the Kh channels of one K part)
    const size_t half_plane = (size_t)NV * 16;             // one K half of one K step, all voxels
    const size_t slab_one = (size_t)NV * Kh * 4;           // hi or lo
    uint32_t* occs = reinterpret_cast<uint32_t*>(gsm + 2 * slab_one);
    unsigned char* bst = gsm + g.slab_bytes;
    uint32_t* wmask = reinterpret_cast<uint32_t*>(
        bst + (g.ball ? (size_t)KV : (size_t)2 * g.bgroup) * g.bstage_bytes);   // after the B region
    int* dlist = reinterpret_cast<int*>(wmask + KV * Np);   // [nd][dlist KV][uniform KV][slab offset KV]
    uint64_t* mbar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(dlist) +
                                                 (((size_t)(3 * KV + 1) * 4 + 7) & ~(size_t)7));
    uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 2 * S);
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(gsm);
    const uint32_t bbase = sbase + (uint32_t)g.slab_bytes;
    const uint32_t mb0 = (uint32_t)__cvta_generic_to_shared(mbar);

    for (int i = tid; i < KV * Np; i += kGThreads) wmask[i] = a.wmask[i];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"((uint32_t)__cvta_generic_to_shared(tslot)), "r"((uint32_t)g.tcols_slab));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(mb0 + 8u * i, kGThreads);
            mbar_init(mb0 + 8u * (S + i), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < 3 * KV + 1; i += kGThreads) dlist[i] = a.dinfo[i];
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const int nd = dlist[0];
    const int* dl = dlist + 1;
    const int* duni = dlist + 1 + KV;
    const int* dsoff = dlist + 1 + 2 * KV;

    // ---- stage the neighbourhood's channels of K part `part` (joins the cp.async group of the
    // first B load): one slab row (sx, sy) per warp iteration, lanes over its SZ voxels x 16-byte
    // chunks; the occupancy masks with the first part
    auto fill_slab = [&](int part) {
        const int cpv = Kh / 4;                              // 16-byte chunks per voxel (2, 4, 6 or 8)
        const int xs0 = x - kg.hx, ys0 = y0 - kg.hy, zs0 = z0 - kg.hz;
        const int lane = tid & 31;
        for (int r = warp; r < g.SX * SY; r += kGThreads / 32) {
            const int sx = r / SY, sy = r - (r / SY) * SY;
            const int qx = xs0 + sx, qy = ys0 + sy;
            const bool rok = qx >= 0 && qx < gx.X && qy >= 0 && qy < gx.Y;
            const size_t rowv = (size_t)b * gx.V + ((size_t)(rok ? qx : 0) * gx.Y + (rok ? qy : 0)) * gx.Z;
            const size_t rowq = rowv * Kp + (size_t)part * Kh;
            for (int j = lane; j < SZ * cpv; j += 32) {
                const int sz = j / cpv, c = j - sz * cpv;
                const int qz = zs0 + sz;
                const bool ok = rok && qz >= 0 && qz < gx.Z;
                const size_t q = ok ? rowq + (size_t)qz * Kp + 4 * c : 0;
                const int v = r * SZ + sz;
                const uint32_t off = (uint32_t)(((c >> 1) * 2 + (c & 1)) * half_plane + (size_t)v * 16);
                cp16(sbase + off, a.xhi + q, ok);
                cp16(sbase + (uint32_t)slab_one + off, a.xlo + q, ok);
            }
            if (part == 0)
                for (int sz = lane; sz < SZ; sz += 32) {
                    const int qz = zs0 + sz;
                    const bool ok = rok && qz >= 0 && qz < gx.Z;
                    cp4(sbase + (uint32_t)(2 * slab_one) + 4u * (uint32_t)(r * SZ + sz), a.occ + (ok ? rowv + qz : 0), ok);
                }
        }
    };
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(Np >> 3) << 17) | ((uint32_t)(kGM >> 4) << 24);
    const uint32_t idesc2 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)((2 * Np) >> 3) << 17) | ((uint32_t)(kGM >> 4) << 24);
    const uint32_t lbo_a = (uint32_t)half_plane, sbo_a = (uint32_t)(SZ * 16);
    const uint64_t dA0 = umma_sdesc(sbase, lbo_a, sbo_a), dB0 = umma_sdesc(bbase);
    const uint64_t kA = (uint64_t)(2 * half_plane >> 4), kB = (uint64_t)(2 * Np * 32 >> 4);
    const size_t B_part = (size_t)2 * Np * Kh;              // floats of one offset's B for one part

    if (nd > 0 && g.ball) {
        // all B_delta resident: one async group (slab + every B), then every MMA back to back and
        // a single commit -- no per-offset synchronisation
        fill_slab(0);
        for (int j = 0; j < nd; ++j) {
            const uint32_t base = bbase + (uint32_t)(j * g.bstage_bytes);
            const float* bh = a.bhi + (size_t)dl[j] * 2 * Np * Kp;
            for (int c = tid; c < 2 * Np * Kp / 4; c += kGThreads) cp16(base + 16u * c, bh + 4 * c, true);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncthreads();
        if (warp == 0) {   // converged warp: MMAs issued through elect.sync
            tc_fence_after();
            for (int it = 0; it < nd; ++it) {
                const uint64_t dAh = dA0 + (uint64_t)((uint32_t)(dsoff[dl[it]] * 16) >> 4);
                const uint64_t dBc = dB0 + (uint64_t)((uint32_t)(it * g.bstage_bytes) >> 4);
                const uint64_t dAl = dAh + (uint64_t)(slab_one >> 4);
                const uint32_t td = tmem + (uint32_t)((it % g.nacc) * 2 * Np);
                for (int ks = 0; ks < Kp / 8; ++ks) {   // A_hi.[W_hi|W_lo], then A_lo.W_hi
                    umma_tf32(td, dAh + ks * kA, dBc + ks * kB, idesc2, (it >= g.nacc || ks != 0) ? 1u : 0u);
                    umma_tf32(td, dAl + ks * kA, dBc + ks * kB, idesc, 1u);
                }
            }
            umma_commit(mb0 + 8u * S);
        }
        mbar_wait(mb0 + 8u * S, 0u);
        tc_fence_after();
    } else if (nd > 0) {
        // per K part: two stages, each holding the B of GD consecutive offsets (this part's K
        // steps of each): group j+1 streams in while the MMAs of group j run; the first group of
        // a part also carries the part's slab. `gi` counts groups over both parts (stage and
        // barrier phase).
        const int GD = g.bgroup;
        const int ngrp = (nd + GD - 1) / GD;
        const size_t gstage = (size_t)GD * g.bstage_bytes;
        auto load_grp = [&](int st, int grp, int part) {
            const uint32_t base = bbase + (uint32_t)(st * gstage);
            for (int j = 0; j < GD && grp * GD + j < nd; ++j) {
                const int d = dl[grp * GD + j];
                const float* bh = a.bhi + (size_t)d * 2 * Np * Kp + (size_t)part * B_part;
                const uint32_t sb = base + (uint32_t)(j * g.bstage_bytes);
                for (int c = tid; c < (int)(B_part / 4); c += kGThreads) cp16(sb + 16u * c, bh + 4 * c, true);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        int gi = 0;
        for (int part = 0; part < g.kparts; ++part) {
            fill_slab(part);
            load_grp(gi & 1, 0, part);
            for (int it = 0; it < ngrp; ++it, ++gi) {
                const int st = gi & 1;
                asm volatile("cp.async.wait_group 0;" ::: "memory");   // this thread's share of group gi
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(mb0 + 8u * st);
                if (warp == 0) {   // converged warp: MMAs issued through elect.sync
                    mbar_wait(mb0 + 8u * st, (uint32_t)((gi >> 1) & 1));
                    tc_fence_after();
                    for (int j = 0; j < GD && it * GD + j < nd; ++j) {
                        const int di = it * GD + j;
                        // descriptors differ only in the start-address field (16-byte units)
                        const uint64_t dAh = dA0 + (uint64_t)((uint32_t)(dsoff[dl[di]] * 16) >> 4);
                        const uint64_t dBc = dB0 + (uint64_t)((uint32_t)(st * gstage + (size_t)j * g.bstage_bytes) >> 4);
                        const uint64_t dAl = dAh + (uint64_t)(slab_one >> 4);
                        const uint32_t td = tmem + (uint32_t)((di % g.nacc) * 2 * Np);
                        for (int ks = 0; ks < Kh / 8; ++ks) {   // A_hi.[W_hi|W_lo], then A_lo.W_hi
                            const uint32_t acc = (part > 0 || di >= g.nacc || ks != 0) ? 1u : 0u;
                            umma_tf32(td, dAh + ks * kA, dBc + ks * kB, idesc2, acc);
                            umma_tf32(td, dAl + ks * kA, dBc + ks * kB, idesc, 1u);
                        }
                    }
                    umma_commit(mb0 + 8u * (S + st));
                }
                // group gi + 1 into the other stage once the MMAs of group gi - 1 retired
                if (it + 1 < ngrp) {
                    if (gi >= 1) mbar_wait(mb0 + 8u * (S + (st ^ 1)), (uint32_t)(((gi - 1) >> 1) & 1));
                    load_grp(st ^ 1, it + 1, part);
                }
            }
            // every MMA of this part retired: the slab and both stages are free again
            mbar_wait(mb0 + 8u * (S + ((gi - 1) & 1)), (uint32_t)(((gi - 1) >> 1) & 1));
            if (gi >= 2) mbar_wait(mb0 + 8u * (S + (gi & 1)), (uint32_t)(((gi - 2) >> 1) & 1));
            tc_fence_after();
        }
    } else {
        fill_slab(0);
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncthreads();   // occupancy slab visible
    }

    // ---- epilogue: TMEM lane m = this thread's M row = (y0 + m/8, z0 + m%8)
    const int yy = tid >> 3, zz = tid & 7;
    const int py = y0 + yy, pz = z0 + zz;
    const bool pin = py < gy.Y && pz < gy.Z;
    if (nd > 0) __syncthreads();   // every thread's occupancy slab writes are visible
    uint64_t supm = 0;
    const uint64_t allm = c_out >= 64 ? ~0ull : ((1ull << c_out) - 1ull);
    if (pin)
        for (int d = 0; d < KV; ++d) {
            const uint32_t nb = occs[dsoff[d] + yy * SZ + zz];
            if (!nb) continue;
            if (duni[d]) {
                if (nb & wmask[d * Np]) supm = allm;
            } else {
                for (int oc = 0; oc < c_out; ++oc)
                    if (nb & wmask[d * Np + oc]) supm |= 1ull << oc;
            }
            if (supm == allm) break;
        }
    const int64_t p = ((int64_t)x * gy.Y + py) * gy.Z + pz;
    for (int c0 = 0; c0 < Np; c0 += 16) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.0f;
        for (int ai = 0; ai < min(g.nacc, nd); ++ai) {   // sum the accumulators, both halves of each
            float u[16], w2[16];
            tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(ai * 2 * Np + c0), u);
            tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(ai * 2 * Np + Np + c0), w2);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += u[i] + w2[i];
        }
        if (!pin) continue;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int oc = c0 + i;
            if (oc >= c_out) break;
            const bool sup = (supm >> oc) & 1ull;
            const float bv = a.bias ? __ldg(&a.bias[oc]) : 0.0f;
            a.pre[((size_t)b * c_out + oc) * gy.V + p] = sup ? v[i] + bv : __uint_as_float(kAbsent);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"((uint32_t)g.tcols_slab));
}

// Support size and score-digit histogram of each (b, oc) buffer (the scatter variant fuses this
// into its epilogue): one block per slice of a segment, shared-memory histogram.
__global__ void __launch_bounds__(256) pre_hist_kernel(FwdArgs a, int64_t V, int splits) {
    __shared__ uint32_t h[kSelBins];
    __shared__ uint32_t sm[33];
    const int64_t s = blockIdx.x / splits;
    const int j = (int)(blockIdx.x - s * splits);
    const int64_t per = (V + splits - 1) / splits;
    const int64_t lo = j * per, hi = min(V, lo + per);
    for (int i = threadIdx.x; i < kSelBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const float* P = a.pre + s * V;
    uint32_t cnt = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const uint32_t bits = __float_as_uint(P[i]);
        if (bits == kAbsent) continue;
        ++cnt;
        if (a.attn != SPC_ATTN_NONE) atomicAdd(&h[score_bits(bits, a.attn) >> 21], 1u);
    }
    __syncthreads();
    if (a.attn != SPC_ATTN_NONE)
        for (int i = threadIdx.x; i < kSelBins; i += blockDim.x)
            if (h[i]) atomicAdd(&a.hist[s * kSelBins + i], h[i]);
    const uint32_t tot = block_sum(cnt, sm);
    if (threadIdx.x == 0 && tot) atomicAdd(&a.seg_count[s], (unsigned long long)tot);
}

cudaError_t launch_conv_gemm(const Geo& gx, const Geo& gy, const KGeo& kg, const GemmPlan& g, const GemmArgs& ga,
                             const FwdArgs& a, cudaStream_t s) {
    const size_t nvox = (size_t)gx.B * gx.V;
    cudaMemsetAsync(ga.bhi, 0, (size_t)2 * g.KV * g.Np * g.Kp * sizeof(float), s);
    cudaMemsetAsync(ga.wmask, 0, (size_t)g.KV * g.Np * sizeof(uint32_t), s);
    // tiled densify when a band of rows fits shared memory (bands of up to 256 voxels)
    const int ny = std::max(1, std::min(gx.Y, 256 / std::max(gx.Z, 1)));
    const size_t dz_smem = (size_t)ny * gx.Z * g.Kp * 8 + (size_t)ny * gx.Z * 4;
    if (ga.xrow && dz_smem <= 100 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(gemm_densify_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)dz_smem);
        if (e != cudaSuccess) return e;
        SPC_PHASE("gemm_densify", s, 1);
        const int64_t tiles = gx.B * gx.X * (int64_t)((gx.Y + ny - 1) / ny);
        gemm_densify_tile_kernel<<<(unsigned)tiles, 256, dz_smem, s>>>(gx, g.Kp, ny, ga.xkeys, ga.xvals, ga.xrow, ga.xhi,
                                                                      ga.xlo, ga.occ);
    } else {
        cudaMemsetAsync(ga.xhi, 0, nvox * g.Kp * sizeof(float), s);
        cudaMemsetAsync(ga.xlo, 0, nvox * g.Kp * sizeof(float), s);
        cudaMemsetAsync(ga.occ, 0, nvox * sizeof(uint32_t), s);
        SPC_PHASE("gemm_densify", s, 1);
        gemm_densify_kernel<<<num_sms() * 8, 256, 0, s>>>(gx, g.Kp, ga.xkeys, ga.xvals, ga.x_nnz_dev, ga.x_nnz, ga.xhi, ga.xlo,
                                                  ga.occ);
    }
    {
        SPC_PHASE("gemm_wprep", s, 1);
        gemm_wprep_kernel<<<32, 256, 0, s>>>(kg, (int)gx.C, g.Kp, g.Np, ga.wkeys, ga.wvals, ga.nw, ga.bhi,
                                             ga.wmask);
    }
    {
        SPC_PHASE("gemm_dinfo", s, 1);
        gemm_dinfo_kernel<<<1, 32, 0, s>>>(kg, (int)gy.C, g.Np, g.SY, g.SZ, ga.wmask, ga.dinfo);
    }
    cudaError_t e;
    {
        SPC_PHASE("conv_gemm", s, 1);
        GemmArgs gg = ga;
        gg.pre = a.pre;
        gg.bias = a.bias;
        if (g.slab) {
            e = cudaFuncSetAttribute(conv_gemm_slab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.slab_smem);
            if (e != cudaSuccess) return e;
            conv_gemm_slab_kernel<<<(unsigned)(gx.B * gy.X * g.nty * g.ntz), kGThreads, g.slab_smem, s>>>(gx, gy, kg, g, gg);
        } else {
            e = cudaFuncSetAttribute(conv_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem);
            if (e != cudaSuccess) return e;
            conv_gemm_kernel<<<(unsigned)(gx.B * g.ntile), kGThreads, g.smem, s>>>(gx, gy, kg, g, gg);
        }
    }
    {
        const int64_t nseg = gy.B * gy.C;
        const int splits = (int)std::max<int64_t>(1, std::min<int64_t>(256, (4 * num_sms() + nseg - 1) / nseg));
        SPC_PHASE("pre_hist", s, 1);
        pre_hist_kernel<<<(unsigned)(nseg * splits), 256, 0, s>>>(a, gy.V, splits);
    }
    return cudaGetLastError();
}

}  // namespace spc

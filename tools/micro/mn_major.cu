// Micro-test (round-2 design input for a tensor-core weight gradient): does tcgen05.mma
// kind::tf32 accept an MN-major A operand (instruction-descriptor bit 15), and which of the
// descriptor's two byte offsets is the stride between MN-adjacent core matrices?
// A: M = 128 x K = 8, MN-major, no swizzle: core matrix = 8 K-rows of 16 bytes (4 consecutive M
// elements each), M-adjacent core matrices 128 bytes apart. B: N = 32 x K = 8, K-major canonical
// (as in conv_gemm.cu). D = A.B (fp32, TMEM) is compared with a host reference for both
// (LBO, SBO) assignments.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o mn_major tools/micro/mn_major.cu && ./mn_major
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((a >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}

constexpr int M = 128, N = 32, K = 8;

__global__ void k(const float* A, const float* B, float* D, uint32_t lbo_a, uint32_t sbo_a, int a_mn) {
    __shared__ __align__(1024) float sa[M * K];
    __shared__ __align__(1024) float sb[N * K];
    __shared__ uint32_t slot;
    __shared__ uint64_t mbar;
    const int tid = threadIdx.x, warp = tid >> 5;
    // A(m, k): MN-major core matrices: offset (m / 4) * 128 B + k * 16 B + (m % 4) * 4 B
    //          K-major canonical (a_mn == 0): (m / 8) * 256 B + (k / 4) * 128 B + (m % 8) * 16 B + (k % 4) * 4 B
    for (int i = tid; i < M * K; i += blockDim.x) {
        const int m = i / K, kk = i % K;
        const int off = a_mn ? (m / 4) * 32 + kk * 4 + (m % 4) : (m / 8) * 64 + (kk / 4) * 32 + (m % 8) * 4 + (kk % 4);
        sa[off] = A[m * K + kk];
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int n = i / K, kk = i % K;
        sb[(n / 8) * 64 + (kk / 4) * 32 + (n % 8) * 4 + (kk % 4)] = B[n * K + kk];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&slot)), "r"(32));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    const uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    if (a_mn) idesc |= 1u << 15;   // transpose A: MN-major
    if (warp == 0) {
        const uint64_t da = a_mn ? sdesc((uint32_t)__cvta_generic_to_shared(sa), lbo_a, sbo_a)
                                 : sdesc((uint32_t)__cvta_generic_to_shared(sa), 128, 256);
        const uint64_t db = sdesc((uint32_t)__cvta_generic_to_shared(sb), 128, 256);
        asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                     :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0));
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" :: "r"(mb) : "memory");
    }
    asm volatile("{\n\t.reg .pred P1;\nW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W%=;\n\t}" :: "r"(mb) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    // lane = row (warp w owns TMEM lanes 32w..32w+31), 32 columns
    uint32_t r[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                   "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                   "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int c = 0; c < 32; ++c) D[tid * N + c] = __uint_as_float(r[c]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(32));
}

int main(int argc, char** argv) {
    std::vector<float> A(M * K), B(N * K), D(M * N), R(M * N);
    const bool probe = argc > 1;   // A(m, k) = m + 1000 k, B(n, k) = (k == n % 8): D(m, n) = A(m, n % 8)
    for (int i = 0; i < M * K; ++i) A[i] = probe ? (float)(i / K + 1000 * (i % K)) : (float)((i * 37 % 17) - 8) / 8.0f;
    for (int i = 0; i < N * K; ++i) B[i] = probe ? ((i % K) == (i / K) % 8 ? 1.0f : 0.0f) : (float)((i * 11 % 13) - 6) / 4.0f;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int kk = 0; kk < K; ++kk) s += (double)A[m * K + kk] * B[n * K + kk];
            R[m * N + n] = (float)s;
        }
    float *dA, *dB, *dD;
    cudaMalloc(&dA, 4 * M * K);
    cudaMalloc(&dB, 4 * N * K);
    cudaMalloc(&dD, 4 * M * N);
    cudaMemcpy(dA, A.data(), 4 * M * K, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), 4 * N * K, cudaMemcpyHostToDevice);
    struct Case { int mn; uint32_t lbo, sbo; char name[96]; };
    std::vector<Case> cases;
    cases.push_back({0, 128, 256, "K-major A (control)"});
    const uint32_t offs[] = {0, 16, 64, 128, 256, 512, 1024, 2048};
    for (uint32_t l : offs)
        for (uint32_t s2 : offs) {
            Case c{1, l, s2, ""};
            snprintf(c.name, sizeof(c.name), "MN-major A, LBO = %u, SBO = %u", l, s2);
            cases.push_back(c);
        }
    for (auto& c : cases) {
        cudaMemset(dD, 0, 4 * M * N);
        k<<<1, 128>>>(dA, dB, dD, c.lbo, c.sbo, c.mn);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, 4 * M * N, cudaMemcpyDeviceToHost);
        int bad = 0;
        double maxerr = 0;
        for (int i = 0; i < M * N; ++i) {
            const double err = std::fabs((double)D[i] - R[i]);
            maxerr = err > maxerr ? err : maxerr;
            bad += err > 1e-6;
        }
        if (bad < M * N / 2 || c.mn == 0)
            printf("%-52s err=%s mismatches=%d/%d max|err|=%.3g\n", c.name, cudaGetErrorString(e), bad, M * N, maxerr);
        if (probe && bad < M * N / 2)
            for (int m = 0; m < 12; ++m) {
                printf("  m=%3d:", m);
                for (int n = 0; n < 8; ++n) printf(" %7.0f", D[m * N + n]);
                printf("\n");
            }
        if (e != cudaSuccess) return 1;
    }
    return 0;
}

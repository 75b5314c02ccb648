// Microbenchmark: throughput of back-to-back tcgen05.mma.kind::tf32 (cta_group::1, M=128) from
// shared-memory operands in the canonical K-major no-swizzle layout, for several N.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((a >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) | ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
template <int N>
__global__ void k(long long* out, int reps, int nacc) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t slot;
    __shared__ uint64_t mbar;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.0f;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(&slot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    uint32_t mb = (uint32_t)__cvta_generic_to_shared(&mbar);
    if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mb)); asm volatile("fence.mbarrier_init.release.cluster;"); }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t tmem = slot;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = 0, t1 = 0;
    if (threadIdx.x < 32) {   // whole warp converged; one elected lane issues
        uint64_t da = sdesc(base, 128, 256), db = sdesc(base + 32768, 128, 256);
        t0 = clock64();
        if (nacc == 1) {
            for (int r = 0; r < reps; ++r) {
                asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" :: "r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(1));
            }
        } else {
            for (int r = 0; r < reps; r += 4) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" :: "r"(tmem + q * N), "l"(da), "l"(db), "r"(idesc), "r"(1));
            }
        }
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" :: "r"(mb) : "memory");
        asm volatile("{\n\t.reg .pred P1;\nW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W%=;\n\t}" :: "r"(mb) : "memory");
        t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(256));
}
template <int N> void run(int reps, int nacc) {
    long long* d; cudaMalloc(&d, 8 * 148);
    cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<N><<<148, 128, 64 * 1024>>>(d, reps, nacc);
    cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, d, 8 * 148, cudaMemcpyDeviceToHost);
    printf("N=%3d nacc=%d reps=%d: %.1f cycles per MMA (block 0), err=%s\n", N, nacc, reps, (double)h[0] / reps, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}
int main() {
    for (int nacc : {1, 4}) { run<32>(2000, nacc); run<64>(2000, nacc); run<128>(2000, nacc); run<256>(1000, 1); }
    return 0;
}

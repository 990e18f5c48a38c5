// Throughput probe: tcgen05.mma kind::i8 dense (K=32) vs .sp 2:4 (K=64 logical) on one CTA,
// M=128, N=256, operands resident in shared memory (values irrelevant for the rate).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(const void *tile) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_u32(tile) >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc_i8(bool sparse, int m, int n) {
    return (sparse ? (1u << 2) : 0u) | (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(m >> 4) << 24);
}

template <bool kSparse>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, unsigned long long *cycles) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_base;
    __shared__ uint64_t bar;
    unsigned char *a = smem, *b = smem + 32768;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = 0x01010101u;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tmem_base;
    const uint32_t tacc = tmem, tmeta = tmem + 256;          // metadata columns 256..
    // metadata: every nibble 0x4 = keep elements (0,1) of each group of 4
    {
        const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + 256;
        uint32_t v0 = 0x44444444u, v1 = 0x44444444u, v2 = 0x44444444u, v3 = 0x44444444u;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v0), "r"(v1), "r"(v2), "r"(v3) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        const uint32_t id = idesc_i8(kSparse, 128, 256);
        const uint64_t da = sw128_desc(a), db = sw128_desc(b);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (kSparse) {
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%5], %3, p;\n\t}"
                        ::"r"(tacc), "l"(da + 2 * k), "l"(db + 4 * (k & 1)), "r"(id), "r"(1), "r"(tmeta) : "memory");
                } else {
                    asm volatile(
                        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                        ::"r"(tacc), "l"(da + 2 * k), "l"(db + 2 * k), "r"(id), "r"(1) : "memory");
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
        long long t1 = clock64();
        cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

extern "C" int run(int sparse, int iters, int blocks, float *ms, double *cyc_per_mma) {
    unsigned long long *d;
    cudaMalloc(&d, sizeof(unsigned long long) * blocks);
    auto k = sparse ? rate_kernel<true> : rate_kernel<false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    k<<<blocks, 128, 65536>>>(4, d);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<blocks, 128, 65536>>>(iters, d);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    cudaEventElapsedTime(ms, a, b);
    unsigned long long h = 0;
    cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
    *cyc_per_mma = (double)h / (4.0 * iters);
    cudaFree(d);
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    e = cudaGetLastError();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}

// Correctness probe for tcgen05.mma.sp kind::i8 (2:4): one MMA, M=128, N=256, K=64 logical.
// Host passes the compressed A (128 x 32 B), B (256 x 64 B), and per-row metadata (2 words);
// the kernel stages A/B in SW128 K-major shared memory, metadata in TMEM (tcgen05.st), runs one
// MMA and returns C (128 x 256 int32).  dense=1 runs the dense K=32 MMA on A (128x32), B (256x32).
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
__host__ __device__ constexpr uint32_t idesc_i8(bool sparse, int m, int n, bool sa, bool sb) {
    return (sparse ? (1u << 2) : 0u) | (2u << 4) | ((sa ? 1u : 0u) << 7) | ((sb ? 1u : 0u) << 10) |
           ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
// byte (row r, k) of a SW128 K-major tile with 128-byte rows
__device__ __forceinline__ int sw128_off(int r, int k) { return r * 128 + ((((k >> 4) ^ (r & 7)) << 4) | (k & 15)); }

__global__ void check_kernel(const int8_t *A, int a_bytes, const int8_t *B, int b_bytes, const uint32_t *meta,
                             int dense, int *C) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_base;
    __shared__ uint64_t bar;
    unsigned char *sa = smem, *sb = smem + 16384;
    for (int i = threadIdx.x; i < 16384 + 32768; i += blockDim.x) smem[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < 128 * a_bytes; i += blockDim.x) sa[sw128_off(i / a_bytes, i % a_bytes)] = A[i];
    for (int i = threadIdx.x; i < 256 * b_bytes; i += blockDim.x) sb[sw128_off(i / b_bytes, i % b_bytes)] = B[i];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
    const uint32_t tmem = tmem_base, tacc = tmem, tmeta = tmem + 256;
    {
        const int row = 32 * warp + lane;
        const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + 256;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(meta[2 * row]), "r"(meta[2 * row + 1]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        const uint64_t da = sw128_desc(sa), db = sw128_desc(sb);
        if (dense) {
            const uint32_t id = idesc_i8(false, 128, 256, true, true);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(tacc), "l"(da), "l"(db), "r"(id), "r"(0) : "memory");
        } else {
            const uint32_t id = idesc_i8(true, 128, 256, true, true);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%5], %3, p;\n\t}"
                         ::"r"(tacc), "l"(da), "l"(db), "r"(id), "r"(0), "r"(tmeta) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int c0 = 0; c0 < 256; c0 += 32) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int row = 32 * warp + lane;
        for (int k = 0; k < 32; ++k) C[row * 256 + c0 + k] = (int)v[k];
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

extern "C" int run(const int8_t *hA, int a_bytes, const int8_t *hB, int b_bytes, const uint32_t *hmeta, int dense, int *hC) {
    int8_t *A, *B; uint32_t *M; int *C;
    cudaMalloc(&A, 128 * a_bytes); cudaMalloc(&B, 256 * b_bytes); cudaMalloc(&M, 128 * 8); cudaMalloc(&C, 128 * 256 * 4);
    cudaMemcpy(A, hA, 128 * a_bytes, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, 256 * b_bytes, cudaMemcpyHostToDevice);
    cudaMemcpy(M, hmeta, 128 * 8, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 32768);
    check_kernel<<<1, 128, 16384 + 32768>>>(A, a_bytes, B, b_bytes, M, dense, C);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(hC, C, 128 * 256 * 4, cudaMemcpyDeviceToHost);
    cudaFree(A); cudaFree(B); cudaFree(M); cudaFree(C);
    return 0;
}

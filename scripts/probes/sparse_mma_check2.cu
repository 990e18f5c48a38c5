// Probe 2: four sparse MMAs (K = 256 logical) accumulating; metadata either written by tcgen05.st
// (mode 0) or copied from shared memory by tcgen05.cp.128x256b (mode 1) from a no-swizzle K-major
// core-matrix layout: core matrix (8 rows x 16 B) at ((row/8)*2 + chunk)*128 B, LBO=128 B, SBO=256 B.
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
__device__ __forceinline__ uint64_t plain_desc(const void *tile, unsigned lbo, unsigned sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_u32(tile) >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;                                                 // layout type 0: no swizzle
}
__host__ __device__ constexpr uint32_t idesc_i8(bool sparse, int m, int n) {
    return (sparse ? (1u << 2) : 0u) | (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ int sw128_off(int r, int k) { return r * 128 + ((((k >> 4) ^ (r & 7)) << 4) | (k & 15)); }

__global__ void check_kernel(const int8_t *A, const int8_t *B, const uint32_t *meta, int mode, unsigned lbo, unsigned sbo, int *C) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ uint32_t tmem_base;
    __shared__ uint64_t bar;
    unsigned char *sa = smem, *sb = smem + 16384, *se = smem + 16384 + 65536;   // A 16K, B 2 x 32K, E 4K
    for (int i = threadIdx.x; i < 16384 + 65536 + 4096; i += blockDim.x) smem[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < 128 * 128; i += blockDim.x) sa[sw128_off(i / 128, i % 128)] = A[i];
    for (int i = threadIdx.x; i < 256 * 256; i += blockDim.x) {
        const int r = i / 256, k = i % 256;
        sb[(k / 128) * 32768 + sw128_off(r, k % 128)] = B[i];
    }
    // metadata rows: 32 bytes per row (4 MMAs x 8 B) in core-matrix order
    for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) {
        const int r = i / 32, b = i % 32;
        const unsigned char v = reinterpret_cast<const unsigned char *>(meta)[r * 32 + b];
        se[((r / 8) * 2 + b / 16) * 128 + (r % 8) * 16 + (b % 16)] = v;
    }
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
    if (mode == 0) {
        const int row = 32 * warp + lane;
        const uint32_t taddr = tmem + ((uint32_t)(32 * warp) << 16) + 256;
        const uint32_t *m = meta + row * 8;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                     ::"r"(taddr), "r"(m[0]), "r"(m[1]), "r"(m[2]), "r"(m[3]), "r"(m[4]), "r"(m[5]), "r"(m[6]), "r"(m[7]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        if (mode == 1) {
            const uint64_t de = plain_desc(se, lbo, sbo);
            asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmeta), "l"(de) : "memory");
        }
        const uint32_t id = idesc_i8(true, 128, 256);
        const uint64_t da = sw128_desc(sa);
        for (int k = 0; k < 4; ++k) {
            const uint64_t db = sw128_desc(sb + (k / 2) * 32768) + 4 * (k % 2);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.sp.cta_group::1.kind::i8 [%0], %1, %2, [%5], %3, p;\n\t}"
                         ::"r"(tacc), "l"(da + 2 * k), "l"(db), "r"(id), "r"(k), "r"(tmeta + 2 * k) : "memory");
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

extern "C" int run(const int8_t *hA, const int8_t *hB, const uint32_t *hmeta, int mode, unsigned lbo, unsigned sbo, int *hC) {
    int8_t *A, *B; uint32_t *M; int *C;
    cudaMalloc(&A, 128 * 128); cudaMalloc(&B, 256 * 256); cudaMalloc(&M, 128 * 32); cudaMalloc(&C, 128 * 256 * 4);
    cudaMemcpy(A, hA, 128 * 128, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, 256 * 256, cudaMemcpyHostToDevice);
    cudaMemcpy(M, hmeta, 128 * 32, cudaMemcpyHostToDevice);
    const int smem = 16384 + 65536 + 4096;
    cudaFuncSetAttribute(check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    check_kernel<<<1, 128, smem>>>(A, B, M, mode, lbo, sbo, C);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(hC, C, 128 * 256 * 4, cudaMemcpyDeviceToHost);
    cudaFree(A); cudaFree(B); cudaFree(M); cudaFree(C);
    return 0;
}

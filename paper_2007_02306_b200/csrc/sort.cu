// sort.cu -- spatial ordering used by mesh staging (triangles) and construction (images).
//
// Not part of the paper's arithmetic: a RICI is a sum over triangles, so the order in
// which triangles are visited, and the order in which images are built, cannot change
// any count.  Ordering only makes consecutive triangles (a chunk) and consecutive images
// (a CTA's group) spatially compact, which is what makes the exact bounding-sphere cull
// in generate.cu effective for arbitrarily ordered inputs.
//
// Method: counting sort of points by an 18-bit cell key (6 bits per axis over the points'
// bounding box; Hilbert order, or Morton with -DRICI_SORT_HILBERT=0): histogram (atomics),
// three-pass exclusive scan, scatter.
#include <algorithm>

#include "rici_internal.cuh"

namespace rici {
namespace {

constexpr int kCellBits = 6;
constexpr int kCells = 1 << (3 * kCellBits);

__device__ __forceinline__ int ordered(float x) {
    int i = __float_as_int(x);
    return i >= 0 ? i : (i ^ 0x7fffffff);
}
__device__ __forceinline__ float unordered(int i) { return __int_as_float(i >= 0 ? i : (i ^ 0x7fffffff)); }

__global__ void bbox_init_kernel(int *box) {
    if (threadIdx.x < 3) box[threadIdx.x] = 0x7fffffff;
    else if (threadIdx.x < 6) box[threadIdx.x] = (int)0x80000000;
}

__global__ void __launch_bounds__(256)
bbox_kernel(const float *__restrict__ pts, int stride, int64_t n, int *__restrict__ box) {
    int lo[3] = {0x7fffffff, 0x7fffffff, 0x7fffffff};
    int hi[3] = {(int)0x80000000, (int)0x80000000, (int)0x80000000};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        for (int a = 0; a < 3; ++a) {
            float v = pts[i * stride + a];
            if (!isfinite(v)) continue;
            int o = ordered(v);
            lo[a] = min(lo[a], o);
            hi[a] = max(hi[a], o);
        }
    }
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = min(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
            hi[a] = max(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
        if ((threadIdx.x & 31) == 0) { atomicMin(box + a, lo[a]); atomicMax(box + 3 + a, hi[a]); }
    }
}

#ifndef RICI_SORT_HILBERT
#define RICI_SORT_HILBERT 1
#endif
#if !RICI_SORT_HILBERT
__device__ __forceinline__ unsigned spread3(unsigned x) {   // 6 bits -> every third bit
    unsigned r = 0;
    for (int b = 0; b < kCellBits; ++b) r |= ((x >> b) & 1u) << (3 * b);
    return r;
}
#endif

// Hilbert index of a cell (Skilling's transpose algorithm, kCellBits bits per axis): unlike the
// Morton (Z) order, consecutive cells along the curve are always face neighbours, so a run of
// 32 surface triangles -- a chunk -- does not jump across the volume between occupied cells
// (C2 model: 19% fewer (image, triangle) pairs tested behind the chunk cull).
__device__ __forceinline__ unsigned hilbert3(unsigned x0, unsigned x1, unsigned x2) {
    unsigned X[3] = {x0, x1, x2};
    const unsigned M = 1u << (kCellBits - 1);
    for (unsigned Q = M; Q > 1; Q >>= 1) {        // inverse undo excess work
        const unsigned P = Q - 1;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if (X[i] & Q) {
                X[0] ^= P;
            } else {
                const unsigned t = (X[0] ^ X[i]) & P;
                X[0] ^= t;
                X[i] ^= t;
            }
        }
    }
    X[1] ^= X[0];                                  // Gray encode
    X[2] ^= X[1];
    unsigned t = 0;
    for (unsigned Q = M; Q > 1; Q >>= 1)
        if (X[2] & Q) t ^= Q - 1;
    X[0] ^= t; X[1] ^= t; X[2] ^= t;
    unsigned h = 0;                                // transpose -> index
    for (int b = kCellBits - 1; b >= 0; --b)
        h = (h << 3) | (((X[0] >> b) & 1u) << 2) | (((X[1] >> b) & 1u) << 1) | ((X[2] >> b) & 1u);
    return h;
}

__device__ __forceinline__ unsigned cell_of(const float *p, const int *box) {
    unsigned c[3];
    for (int a = 0; a < 3; ++a) {
        float lo = unordered(box[a]), hi = unordered(box[3 + a]);
        float ext = hi - lo;
        float t = (ext > 0.f && isfinite(p[a])) ? (p[a] - lo) / ext : 0.f;
        int q = (int)(t * (float)(1 << kCellBits));
        c[a] = (unsigned)min(max(q, 0), (1 << kCellBits) - 1);
    }
#if RICI_SORT_HILBERT
    return hilbert3(c[0], c[1], c[2]);
#else
    return spread3(c[0]) | (spread3(c[1]) << 1) | (spread3(c[2]) << 2);
#endif
}

__global__ void __launch_bounds__(256)
hist_kernel(const float *__restrict__ pts, int stride, int64_t n, const int *__restrict__ box,
            unsigned *__restrict__ cell, int *__restrict__ hist) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned c = cell_of(pts + i * stride, box);
        cell[i] = c;
        atomicAdd(hist + c, 1);
    }
}

// exclusive scan of kCells ints: per-block scans, a scan of the block totals, a fix-up pass
__device__ __forceinline__ int block_exclusive_scan_1024(int v, int *warp_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = warp_tot[lane], wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        warp_tot[lane] = wi - w;                  // exclusive prefix of warp totals
    }
    __syncthreads();
    return incl - v + warp_tot[warp];
}

__global__ void __launch_bounds__(1024) scan_blocks_kernel(int *__restrict__ hist, int *__restrict__ sums) {
    __shared__ int warp_tot[32];
    const int i = blockIdx.x * 1024 + threadIdx.x;
    const int v = hist[i];
    const int ex = block_exclusive_scan_1024(v, warp_tot);
    hist[i] = ex;
    if (threadIdx.x == 1023) sums[blockIdx.x] = ex + v;
}

__global__ void __launch_bounds__(1024) scan_sums_kernel(int *__restrict__ sums, int n) {
    __shared__ int warp_tot[32];
    const int v = threadIdx.x < n ? sums[threadIdx.x] : 0;
    const int ex = block_exclusive_scan_1024(v, warp_tot);
    if (threadIdx.x < n) sums[threadIdx.x] = ex;
}

__global__ void __launch_bounds__(1024) scan_add_kernel(int *__restrict__ hist, const int *__restrict__ sums) {
    hist[blockIdx.x * 1024 + threadIdx.x] += sums[blockIdx.x];
}

__global__ void __launch_bounds__(256)
scatter_kernel(const unsigned *__restrict__ cell, int64_t n, int *__restrict__ offs, int *__restrict__ perm) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        perm[atomicAdd(offs + cell[i], 1)] = (int)i;
}

// Chunk partition inside each superchunk (kSuper * kChunk = 1024 points of the cell order):
// a kd-tree of median splits down to 32-triangle leaves.  Cell order alone makes runs of 32
// that straddle several cells; median splits along each node's longest centroid extent make
// compact leaves, so the chunk spheres -- and the pairs the construction kernel tests behind
// them -- shrink (C2 model: 22% fewer tested pairs).  The superchunks keep their triangle sets.
// One CTA of 1024 threads per full superchunk, one triangle per thread: at each of the five
// levels every node (a 1024 >> l aligned segment) is bitonic-sorted by its longest axis, and
// its halves become the children.  The partial last superchunk keeps the cell order.
constexpr int kKdBlock = 1024;                 // = kSuper * kChunk
__global__ void __launch_bounds__(kKdBlock)
kd_chunks_kernel(const float *__restrict__ pts, int stride, int *__restrict__ order, int64_t nt) {
    static_assert(kKdBlock == 1024, "one thread per triangle of a superchunk");
    __shared__ float xkey[2][kKdBlock];                    // double-buffered exchange (j >= 32)
    __shared__ int xidx[2][kKdBlock];
    __shared__ float wbox[kKdBlock / 32][6];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int64_t base = (int64_t)blockIdx.x * kKdBlock;
    if (base + kKdBlock > nt) return;                      // partial block: keep the cell order
    int iv = order[base + t];
    int buf = 0;
    for (int S = kKdBlock; S > kChunk; S >>= 1) {
        // this node's bounding box: warp reductions, then the warps of the node
        const float *pp = pts + (int64_t)stride * iv;
        const float c[3] = {pp[0], pp[1], pp[2]};
        float lo[3] = {c[0], c[1], c[2]}, hi[3] = {c[0], c[1], c[2]};
#pragma unroll
        for (int a = 0; a < 3; ++a)
            for (int o = 16; o > 0; o >>= 1) {
                lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
                hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
            }
        if (lane == 0)
            for (int a = 0; a < 3; ++a) { wbox[warp][a] = lo[a]; wbox[warp][3 + a] = hi[a]; }
        __syncthreads();
        const int w0 = (t / S) * (S / 32), nw = S / 32;
        for (int w = w0; w < w0 + nw; ++w)
            for (int a = 0; a < 3; ++a) { lo[a] = fminf(lo[a], wbox[w][a]); hi[a] = fmaxf(hi[a], wbox[w][3 + a]); }
        const float ex = hi[0] - lo[0], ey = hi[1] - lo[1], ez = hi[2] - lo[2];
        float kv = ex >= ey ? (ex >= ez ? c[0] : c[2]) : (ey >= ez ? c[1] : c[2]);
        // bitonic sort of every aligned segment of S (ascending); partners within a warp by
        // shuffle, farther ones through shared memory
        for (int k = 2; k <= S; k <<= 1) {
            const bool up = k == S || (t & k) == 0;
            for (int j = k >> 1; j > 0; j >>= 1) {
                float pk;
                int pi;
                if (j >= 32) {
                    xkey[buf][t] = kv;
                    xidx[buf][t] = iv;
                    __syncthreads();
                    pk = xkey[buf][t ^ j];
                    pi = xidx[buf][t ^ j];
                    buf ^= 1;
                } else {
                    pk = __shfl_xor_sync(0xffffffffu, kv, j);
                    pi = __shfl_xor_sync(0xffffffffu, iv, j);
                }
                const bool lower = (t & j) == 0;           // keep the min iff lower == up
                if (lower == up ? pk < kv : pk > kv) { kv = pk; iv = pi; }
            }
        }
        __syncthreads();                                   // wbox reuse at the next level
    }
    order[base + t] = iv;
}

}  // namespace

// perm[k] = index of the k-th point in cell order (Hilbert curve over 64^3 cells).  pts: n points, `stride` floats apart.
// Workspace is stream-ordered.
cudaError_t spatial_order(const float *d_pts, int stride, int64_t n, int *d_perm, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    cudaError_t e;
    static_assert(kCells % 1024 == 0 && kCells / 1024 <= 1024, "scan layout");
    int *box = nullptr, *hist = nullptr, *sums = nullptr;
    unsigned *cell = nullptr;
    if ((e = cudaMallocAsync((void **)&box, 6 * sizeof(int), s)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync((void **)&hist, kCells * sizeof(int), s)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync((void **)&cell, n * sizeof(unsigned), s)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync((void **)&sums, (kCells / 1024) * sizeof(int), s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(hist, 0, kCells * sizeof(int), s)) != cudaSuccess) return e;
    int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
    bbox_init_kernel<<<1, 32, 0, s>>>(box);
    bbox_kernel<<<blocks, 256, 0, s>>>(d_pts, stride, n, box);
    hist_kernel<<<blocks, 256, 0, s>>>(d_pts, stride, n, box, cell, hist);
    scan_blocks_kernel<<<kCells / 1024, 1024, 0, s>>>(hist, sums);
    scan_sums_kernel<<<1, 1024, 0, s>>>(sums, kCells / 1024);
    scan_add_kernel<<<kCells / 1024, 1024, 0, s>>>(hist, sums);
    scatter_kernel<<<blocks, 256, 0, s>>>(cell, n, hist, d_perm);
    note_launches(7);
    e = cudaGetLastError();
    cudaFreeAsync(box, s);
    cudaFreeAsync(hist, s);
    cudaFreeAsync(cell, s);
    cudaFreeAsync(sums, s);
    return e;
}

// Refine a cell order into kd-tree leaves of 32 inside every full block of 1024 (see above).
cudaError_t kd_refine(const float *d_pts, int stride, int64_t n, int *d_perm, cudaStream_t s) {
    static_assert(kKdBlock == kSuper * kChunk, "a kd block is one superchunk");
    if (n < kKdBlock) return cudaSuccess;
    kd_chunks_kernel<<<(unsigned)(n / kKdBlock), kKdBlock, 0, s>>>(d_pts, stride, d_perm, n);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace rici

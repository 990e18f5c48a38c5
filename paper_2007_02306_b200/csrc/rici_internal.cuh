// rici_internal.cuh -- internal declarations shared by the CUDA translation units
// of librici.so (product path; never includes or links anything from oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rici {

// Triangles are stored in chunks of kChunk, structure-of-arrays inside a chunk:
// tri[(chunk*9 + k)*kChunk + lane], k = 0..8 -> v0.x v0.y v0.z v1.x ... v2.z.
// A warp loads one chunk with 9 fully coalesced 128-byte loads.  (A 48-byte record per triangle
// loaded with three 16-byte loads measured the same: C4 289.4 vs 289.6 ms, r2v.)
constexpr int kChunk = 32;
constexpr int kSuper = 32;   // chunks per superchunk (two-level cull hierarchy)
constexpr int kTriFloatsPerChunk = 9 * kChunk;
// v[0..8] of triangle `lane` of chunk `chunk`
__device__ __forceinline__ void load_triangle(const float *__restrict__ tri, int64_t chunk, int lane, float *v) {
    const float *src = tri + chunk * 9 * kChunk + lane;
#pragma unroll
    for (int c = 0; c < 9; ++c) v[c] = __ldg(src + c * kChunk);
}

struct DeviceMesh {
    int64_t nt = 0;               // triangles
    int64_t n_chunks = 0;         // ceil(nt / kChunk)
    int64_t n_super = 0;          // ceil(n_chunks / kSuper)
    float *tri = nullptr;         // [n_chunks][kTriFloatsPerChunk], triangles in spatial (Hilbert-cell) order
    float4 *sphere = nullptr;     // [n_chunks] bounding sphere (cx, cy, cz, r) of each chunk
    float4 *super_sphere = nullptr;  // [n_super] bounding sphere of each superchunk
    int *order = nullptr;         // [nt] staged slot -> caller triangle index
    int device = 0;
};

// perm[k] = index of the k-th of n points (stride floats apart) in spatial order.
cudaError_t spatial_order(const float *d_pts, int stride, int64_t n, int *d_perm, cudaStream_t s);
// kd-tree leaves of 32 inside every full block of 1024 of a spatial order (sort.cu)
cudaError_t kd_refine(const float *d_pts, int stride, int64_t n, int *d_perm, cudaStream_t s);

// Kernel-launch bookkeeping (rici_launch_count()).
void note_launches(int k);
// Per-kernel event timing (rici_set_kernel_timing): a KernelTimer brackets one API call's
// launches of a timed kernel on stream s.  begin() records the start event (nothing while timing
// is off); end() records the stop event and files the pair; an un-ended timer (an error return
// in between) gives its start event back on destruction, so concurrent calls never pair one
// call's begin with another's end.
cudaEvent_t timing_begin(int kernel, cudaStream_t s);    // nullptr while timing is off
void timing_end(int kernel, cudaStream_t s, cudaEvent_t begin);
void timing_release(cudaEvent_t begin);
struct KernelTimer {
    int kernel;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    KernelTimer(int k, cudaStream_t st) : kernel(k), s(st) { a = timing_begin(k, st); }
    void end() { if (a) { timing_end(kernel, s, a); a = nullptr; } }
    ~KernelTimer() { if (a) timing_release(a); }
    KernelTimer(const KernelTimer &) = delete;
    KernelTimer &operator=(const KernelTimer &) = delete;
};

// Raises a kernel's dynamic shared-memory limit to `bytes` on the current device (once per
// (kernel, device); thread-safe).
cudaError_t ensure_smem(const void *kernel, size_t bytes);

// Largest triangle count the construction work items can address (chunk index << 8 in 31 bits).
constexpr int64_t kMaxTriangles = ((int64_t)1 << 23) * 32;

// a1: de-index + chunk layout + chunk spheres; *d_bad set to 1 on an out-of-range index.
cudaError_t launch_mesh_stage_begin(const float *d_vertices, int64_t nv, const int32_t *d_indices,
                                    int64_t nt, DeviceMesh *m, int *d_bad, float **centroid_out, cudaStream_t s);
cudaError_t launch_mesh_stage_end(const float *d_vertices, int64_t nv, const int32_t *d_indices,
                                  int64_t nt, DeviceMesh *m, float *centroid, cudaStream_t s);

// a2-a8: RICI construction.
cudaError_t launch_generate(const DeviceMesh &m, const float *d_origins, int64_t n, float R,
                            int N, uint16_t *d_out, cudaStream_t s);

// a10: out[k] = CRSS(needles[pairs[k].x], haystack[pairs[k].y]); pairs = nullptr -> (k,k).
cudaError_t launch_crss_pairs(const uint16_t *d_needles, int64_t nn, const uint16_t *d_haystack,
                              int64_t nh, int N, const int64_t *d_pairs, int64_t m,
                              uint64_t *d_out, cudaStream_t s);

// a9 + a11 + a12: count (thresholds != nullptr) or full distances (d_dist != nullptr).
cudaError_t launch_crss_search_tiles(const uint16_t *d_needles, int64_t nn,
                                     const uint16_t *d_haystack, int64_t nh, int N,
                                     const uint64_t *d_thresholds, uint32_t *d_counts,
                                     uint64_t *d_dist, cudaStream_t s, bool early_exit = false);

// a9-a12 on the tensor cores (N = 64): rank counts with the int8 tcgen05 GEMM formulation,
// exact fallback to the SIMT kernel for images outside the int8 guard.
// thr_from_pairs: d_thr is OUTPUT, t_i = CRSS(n_i, h_i) computed in the feature pass (nn <= nh).
// rank_mode: tiles whose pairs are all ruled out by a K-prefix lower bound skip the rest (f1).
cudaError_t launch_crss_count_mma(const uint16_t *d_needles, int64_t nn, const uint16_t *d_haystack, int64_t nh,
                                  uint64_t *d_thr, bool thr_from_pairs, bool rank_mode, uint32_t *d_counts,
                                  cudaStream_t s);

// rici_crss_guard_stats: {needles, needles outside the int8 guard, haystack images, haystack
// images outside it, guard-valid needles that are not 2:4} accumulated on the current device.
cudaError_t read_guard_stats(unsigned long long out[5], bool reset);

// f4: Eq. 8 clutter fraction per oriented point (quadrature of the area inside the support
// cylinder; object_tag [nt] in caller triangle order, device memory).
cudaError_t launch_clutter_fraction(const DeviceMesh &m, const unsigned char *d_tag, const float *d_origins,
                                    int64_t n, float R, int Q, float *d_frac, float *d_area_all, cudaStream_t s);

// Which kernel counts ranks: the tensor-core path when N == 64 and RICI_CRSS_PATH != "simt".
bool use_mma_path(int N);
// Tuning knobs from the environment (read once by each caller into a function-local static).
int env_int(const char *name, int dflt);
double env_double(const char *name, double dflt);

}  // namespace rici

// mesh.cu -- (a1) mesh staging for the construction kernel.
//
// "iterate over each triangle in the scene": the construction kernel streams every
// triangle once per group of images, so the indexed mesh (vertices + index triples, D1) is
// de-indexed once into a device buffer laid out for that stream:
//  * triangles in spatial order (an 18-bit Hilbert cell key of the centroid, counting sort in
//    sort.cu) -- an internal reordering that cannot change any image, counts being sums
//    over triangles; the permutation is kept for per-triangle tags (rici_clutter_fraction);
//  * chunks of 32 triangles, structure-of-arrays inside a chunk, so one warp reads a chunk
//    with nine coalesced 128-byte loads; inside each superchunk the chunks are the leaves of
//    a median-split kd-tree over the centroids (kd_chunks_kernel), so they are compact;
//  * a bounding sphere per chunk and per superchunk (32 chunks) that let the construction
//    and clutter kernels skip triangles that cannot reach a support volume (an exact cull:
//    such triangles add 0).
#include <algorithm>

#include "rici_internal.cuh"

namespace rici {
namespace {

// Validates the index triples and writes each triangle's centroid (the sort key).
__global__ void __launch_bounds__(256)
centroid_kernel(const float *__restrict__ vertices, int64_t nv, const int32_t *__restrict__ indices,
                int64_t nt, float *__restrict__ centroid, int *__restrict__ bad) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += (int64_t)gridDim.x * blockDim.x) {
        float c[3] = {0.f, 0.f, 0.f};
        bool ok = true;
        for (int j = 0; j < 3; ++j) {
            int32_t id = indices[3 * t + j];
            if (id < 0 || (int64_t)id >= nv) { ok = false; continue; }
            for (int a = 0; a < 3; ++a) c[a] += vertices[3 * (int64_t)id + a];
        }
        if (!ok) atomicExch(bad, 1);
        for (int a = 0; a < 3; ++a) centroid[3 * t + a] = c[a] * (1.0f / 3.0f);
    }
}

__global__ void __launch_bounds__(256)
mesh_stage_kernel(const float *__restrict__ vertices, int64_t nv,
                  const int32_t *__restrict__ indices, const int *__restrict__ order, int64_t nt,
                  float *__restrict__ tri, float4 *__restrict__ sphere, int64_t n_chunks) {
    const int lane = threadIdx.x & 31;
    const int64_t chunk = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (chunk >= n_chunks) return;
    int64_t slot = chunk * kChunk + lane;
    const bool real = slot < nt;
    if (!real) slot = chunk * kChunk;         // pad with a copy of lane 0's vertex 0 (degenerate)
    const int64_t t = order[slot];
    float v[9];
    for (int j = 0; j < 3; ++j) {
        int32_t id = indices[3 * t + (real ? j : 0)];
        if (id < 0 || (int64_t)id >= nv) id = 0;  // reported by centroid_kernel
        v[3 * j + 0] = vertices[3 * (int64_t)id + 0];
        v[3 * j + 1] = vertices[3 * (int64_t)id + 1];
        v[3 * j + 2] = vertices[3 * (int64_t)id + 2];
    }
    float *dst = tri + chunk * 9 * kChunk;
#pragma unroll
    for (int k = 0; k < 9; ++k) dst[k * kChunk + lane] = v[k];

    // chunk bounding sphere: bbox centre, max vertex distance
    float lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = fminf(v[a], fminf(v[3 + a], v[6 + a]));
        hi[a] = fmaxf(v[a], fmaxf(v[3 + a], v[6 + a]));
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
            hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
    }
    float c[3] = {0.5f * (lo[0] + hi[0]), 0.5f * (lo[1] + hi[1]), 0.5f * (lo[2] + hi[2])};
    float r2 = 0.f;
    for (int j = 0; j < 3; ++j) {
        float dx = v[3 * j] - c[0], dy = v[3 * j + 1] - c[1], dz = v[3 * j + 2] - c[2];
        r2 = fmaxf(r2, dx * dx + dy * dy + dz * dz);
    }
    for (int o = 16; o > 0; o >>= 1) r2 = fmaxf(r2, __shfl_xor_sync(0xffffffffu, r2, o));
    if (lane == 0) {
        float scale = fmaxf(fabsf(c[0]), fmaxf(fabsf(c[1]), fabsf(c[2])));
        float r = sqrtf(r2) * (1.0f + 1e-5f) + 1e-6f * scale + 1e-30f;   // conservative pad
        sphere[chunk] = make_float4(c[0], c[1], c[2], r);
    }
}

// Superchunk sphere = sphere enclosing its (up to kSuper) chunk spheres; warp per superchunk.
__global__ void __launch_bounds__(256)
super_sphere_kernel(const float4 *__restrict__ sphere, int64_t n_chunks, float4 *__restrict__ sup,
                    int64_t n_super) {
    const int lane = threadIdx.x & 31;
    const int64_t sc = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (sc >= n_super) return;
    int64_t c = sc * kSuper + lane;
    float4 s = sphere[c < n_chunks ? c : sc * kSuper];
    float lo[3] = {s.x - s.w, s.y - s.w, s.z - s.w}, hi[3] = {s.x + s.w, s.y + s.w, s.z + s.w};
    for (int a = 0; a < 3; ++a)
        for (int o = 16; o > 0; o >>= 1) {
            lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
            hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
    float cx = 0.5f * (lo[0] + hi[0]), cy = 0.5f * (lo[1] + hi[1]), cz = 0.5f * (lo[2] + hi[2]);
    float dx = s.x - cx, dy = s.y - cy, dz = s.z - cz;
    float r = sqrtf(dx * dx + dy * dy + dz * dz) + s.w;
    for (int o = 16; o > 0; o >>= 1) r = fmaxf(r, __shfl_xor_sync(0xffffffffu, r, o));
    if (lane == 0) {
        float scale = fmaxf(fabsf(cx), fmaxf(fabsf(cy), fabsf(cz)));
        sup[sc] = make_float4(cx, cy, cz, r * (1.0f + 1e-5f) + 1e-6f * scale + 1e-30f);
    }
}

}  // namespace

// Two phases so the caller's synchronous index check waits only for the validating centroid
// pass: begin() launches it (and allocates the sort keys), end() enqueues the spatial sort and
// the staging kernels after the check has passed, and returns without waiting.  The caller
// owns (and frees) the sort-key buffer begin() allocates.
cudaError_t launch_mesh_stage_begin(const float *d_vertices, int64_t nv, const int32_t *d_indices,
                                    int64_t nt, DeviceMesh *m, int *d_bad, float **centroid_out, cudaStream_t s) {
    m->nt = nt;
    m->n_chunks = (nt + kChunk - 1) / kChunk;
    m->n_super = (m->n_chunks + kSuper - 1) / kSuper;
    *centroid_out = nullptr;
    if (m->n_chunks == 0) return cudaSuccess;
    cudaError_t e;
    float *centroid = nullptr;
    if ((e = cudaMallocAsync((void **)&centroid, sizeof(float) * 3 * nt, s)) != cudaSuccess) return e;
    *centroid_out = centroid;
    if ((e = cudaMallocAsync((void **)&m->order, sizeof(int) * nt, s)) != cudaSuccess) return e;
    int blocks = (int)std::min<int64_t>((nt + 255) / 256, 148 * 8);
    centroid_kernel<<<blocks, 256, 0, s>>>(d_vertices, nv, d_indices, nt, centroid, d_bad);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_mesh_stage_end(const float *d_vertices, int64_t nv, const int32_t *d_indices,
                                  int64_t nt, DeviceMesh *m, float *centroid, cudaStream_t s) {
    if (m->n_chunks == 0) return cudaSuccess;
    cudaError_t e;
    int *order = m->order;
    if ((e = spatial_order(centroid, 3, nt, order, s)) != cudaSuccess) return e;
#ifndef RICI_KD_CHUNKS
#define RICI_KD_CHUNKS 1
#endif
    if (RICI_KD_CHUNKS && (e = kd_refine(centroid, 3, nt, order, s)) != cudaSuccess) return e;
    const int warps = 8;
    int64_t b2 = (m->n_chunks + warps - 1) / warps;
    mesh_stage_kernel<<<(unsigned)b2, 32 * warps, 0, s>>>(d_vertices, nv, d_indices, order, nt, m->tri,
                                                         m->sphere, m->n_chunks);
    int64_t b3 = (m->n_super + warps - 1) / warps;
    super_sphere_kernel<<<(unsigned)b3, 32 * warps, 0, s>>>(m->sphere, m->n_chunks, m->super_sphere, m->n_super);
    note_launches(2);
    return cudaGetLastError();                    // the caller frees centroid (stream-ordered)
}

}  // namespace rici

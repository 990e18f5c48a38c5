// clutter.cu -- (f4) Eq. 8 clutter fraction per oriented point.
//
//     clutter = (A_all - A_object) / A_all
// A_all: surface area of all objects inside the support volume; A_object: the part that
// belongs to the object of interest.  Support volume = the RICI support cylinder,
// r <= R and |beta| <= R/2 (G4, G17).  The paper does not say how the area is measured
// (G17): each triangle is cut into Q x Q congruent sub-triangles on a barycentric grid and a
// sub-triangle counts with area A/Q^2 when its centroid lies inside the volume.
//
// One warp per image.  Candidate triangles come from the same exact hierarchy as the
// construction kernel (superchunk sphere, chunk sphere, then per-triangle sample tests);
// lanes own triangles, per-lane float partial areas are reduced in double.
#include "frame.cuh"
#include "rici_internal.cuh"

namespace rici {
namespace {

__global__ void __launch_bounds__(256)
clutter_kernel(const float *__restrict__ tri, const float4 *__restrict__ sphere, int64_t n_chunks,
               const float4 *__restrict__ super_sphere, int64_t n_super, const int *__restrict__ order,
               int64_t nt, const unsigned char *__restrict__ tag, const float *__restrict__ origins,
               int64_t n, float R, int Q, float *__restrict__ frac, float *__restrict__ area_all) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= n) return;
    const Frame f = make_frame(origins + 6 * i);
    float a_all = 0.f, a_obj = 0.f;
    if (f.valid != 0.f) {
        const float rs = R * 1.1180340f * (1.0f + 1e-5f) + 1e-6f;   // support-cylinder bounding sphere
        const float hr = 0.5f * R, r2 = R * R;
        const float inv_q = 1.0f / (float)Q, inv_q2 = inv_q * inv_q;
        for (int64_t sb = 0; sb < n_super; sb += 32) {
            const int64_t sc_l = sb + lane;
            bool keep = false;
            if (sc_l < n_super) {
                float4 s4 = super_sphere[sc_l];
                float dx = s4.x - f.sx, dy = s4.y - f.sy, dz = s4.z - f.sz, rr = s4.w + rs;
                keep = dx * dx + dy * dy + dz * dz <= rr * rr;
            }
            unsigned sm = __ballot_sync(0xffffffffu, keep);
            while (sm) {
                const int64_t sc = sb + (__ffs(sm) - 1);
                sm &= sm - 1;
                const int64_t c_l = sc * kSuper + lane;
                bool ck = false;
                if (c_l < n_chunks) {                       // chunk sphere vs the support cylinder
                    float4 s4 = sphere[c_l];
                    float dx = s4.x - f.sx, dy = s4.y - f.sy, dz = s4.z - f.sz;
                    float b = fmaf(f.czx, dx, fmaf(f.czy, dy, f.czz * dz));
                    float a2 = fmaxf(dx * dx + dy * dy + dz * dz - b * b, 0.f);
                    float pad = 1e-4f * R + 1e-6f * (fabsf(s4.x) + fabsf(s4.y) + fabsf(s4.z) + s4.w);
                    float ra = R + s4.w + pad;
                    ck = fabsf(b) <= hr + s4.w + pad && a2 <= ra * ra;
                }
                unsigned cm = __ballot_sync(0xffffffffu, ck);
                while (cm) {
                    const int64_t chunk = sc * kSuper + (__ffs(cm) - 1);
                    cm &= cm - 1;
                    const int64_t slot = chunk * kChunk + lane;
                    if (slot >= nt) continue;               // padding of the last chunk
                    float v[9];
                    load_triangle(tri, chunk, lane, v);
                    const float e1x = v[3] - v[0], e1y = v[4] - v[1], e1z = v[5] - v[2];
                    const float e2x = v[6] - v[0], e2y = v[7] - v[1], e2z = v[8] - v[2];
                    const float cx = e1y * e2z - e1z * e2y, cy = e1z * e2x - e1x * e2z, cz = e1x * e2y - e1y * e2x;
                    const float sub = 0.5f * sqrtf(cx * cx + cy * cy + cz * cz) * inv_q2;
                    const float ox = v[0] - f.sx, oy = v[1] - f.sy, oz = v[2] - f.sz;   // Eq. 2
                    int hits = 0;
                    for (int u = 0; u < Q; ++u)
                        for (int w = 0; u + w < Q; ++w)
                            for (int up = 1; up >= 0; --up) {
                                if (!up && u + w >= Q - 1) continue;          // downward sub-triangles
                                const float bu = ((float)u + (up ? 1.f / 3.f : 2.f / 3.f)) * inv_q;
                                const float bw = ((float)w + (up ? 1.f / 3.f : 2.f / 3.f)) * inv_q;
                                const float dx = fmaf(bu, e1x, fmaf(bw, e2x, ox));
                                const float dy = fmaf(bu, e1y, fmaf(bw, e2y, oy));
                                const float dz = fmaf(bu, e1z, fmaf(bw, e2z, oz));
                                const float b = fmaf(f.czx, dx, fmaf(f.czy, dy, f.czz * dz));
                                const float a2 = dx * dx + dy * dy + dz * dz - b * b;
                                hits += (fabsf(b) <= hr) & (a2 <= r2);
                            }
                    const float a = sub * (float)hits;
                    a_all += a;
                    if (tag[order[slot]]) a_obj += a;
                }
            }
        }
    }
    double da = a_all, db = a_obj;
    for (int o = 16; o > 0; o >>= 1) {
        da += __shfl_xor_sync(0xffffffffu, da, o);
        db += __shfl_xor_sync(0xffffffffu, db, o);
    }
    if (lane == 0) {
        frac[i] = da > 0.0 ? (float)((da - db) / da) : 0.f;
        if (area_all) area_all[i] = (float)da;
    }
}

}  // namespace

cudaError_t launch_clutter_fraction(const DeviceMesh &m, const unsigned char *d_tag, const float *d_origins,
                                    int64_t n, float R, int Q, float *d_frac, float *d_area_all, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int warps = 8;
    clutter_kernel<<<(unsigned)((n + warps - 1) / warps), 32 * warps, 0, s>>>(
        m.tri, m.sphere, m.n_chunks, m.super_sphere, m.n_super, m.order, m.nt, d_tag, d_origins, n, R, Q,
        d_frac, d_area_all);
    note_launches(1);
    return cudaGetLastError();
}

}  // namespace rici

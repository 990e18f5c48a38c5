// frame.cuh -- the per-image spin frame (Eq. 1 with the G1 correction),
// shared by the construction kernel (generate.cu) and the clutter-fraction kernel (clutter.cu).
#pragma once
#include <cuda_runtime.h>

namespace rici {
namespace {

struct __align__(16) Frame {
    float sx, sy, sz, valid;      // S_v (Eq. 2); valid = 0 for a zero / non-finite normal (G3)
    float nax, nay, nbx, nbz;     // Eq. 1 with the G1 correction
    float czx, czy, czz, pad;     // T_z = nbx*(nax x + nay y) + nbz z, Eqs. 3-4 composed
};

__device__ __forceinline__ Frame make_frame(const float *o) {
    Frame f;
    f.sx = o[0]; f.sy = o[1]; f.sz = o[2];
    float nx = o[3], ny = o[4], nz = o[5];
    float l2 = nx * nx + ny * ny + nz * nz;
    bool ok = (l2 > 0.f) && isfinite(l2) && isfinite(f.sx) && isfinite(f.sy) && isfinite(f.sz);
    f.valid = ok ? 1.f : 0.f;
    f.pad = 0.f;
    if (!ok) {
        f.nax = 1.f; f.nay = 0.f; f.nbx = 0.f; f.nbz = 1.f; f.czx = f.czy = 0.f; f.czz = 1.f;
        return f;
    }
    float l = sqrtf(l2);
    nx /= l; ny /= l; nz /= l;                       // G3: normalise S_n
    float la2 = nx * nx + ny * ny;
    if (la2 > 0.f) {                                 // Eq. 1: N_a = Normalize[S_nx, S_ny]
        float la = sqrtf(la2);
        f.nax = nx / la; f.nay = ny / la;
    } else {                                         // identity rotation (G2)
        f.nax = 1.f; f.nay = 0.f;
    }
    float s = f.nax * nx + f.nay * ny;               // normal's x after rotation 1 (G1)
    float lb = sqrtf(s * s + nz * nz);
    f.nbx = s / lb; f.nbz = nz / lb;                 // N_b = Normalize[s, S_nz]
    f.czx = f.nbx * f.nax; f.czy = f.nbx * f.nay; f.czz = f.nbz;
    return f;
}

}  // namespace
}  // namespace rici

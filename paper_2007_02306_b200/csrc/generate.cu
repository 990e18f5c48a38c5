// generate.cu -- (a2-a8) RICI construction on sm_100a.
//
// Paper: a RICI pixel counts the intersections of a circle (radius rho_c, at
// height beta_r on the Central Axis) with the scene surface.  It is
// built by iterating over the triangles in three steps:
//   1. project the triangle's vertices into the spin frame (Eqs. 1-5),
//   2. for each layer beta in the triangle's beta-extent, intersect the layer
//      plane with the triangle (segment E0E1), rotate it parallel to x and get
//      the single range [min|E|, max|E|) and, when the x signs differ, the
//      double range [|C|, min|E|) (six steps),
//   3. increment the bins whose circle radius falls in those ranges.
//
// B200 design:
//  * one CTA owns K images (K = 2 at N = 64, 3 CTAs / SM); their 32-bit counters live in
//    shared memory as per-row DIFFERENCE arrays of N+1 columns (column N a sink), so a
//    segment costs 3 branch-free shared reductions (+2 at col(|C|), -1 at col(min), -1 at
//    col(max)) instead of one per covered bin; a per-row prefix scan in the epilogue turns
//    them into counts;
//  * every image's frame is pre-scaled to BIN units (layer r at Z = r, column c's circle at
//    radius c + 1/2), after the translation of Eq. 2;
//  * images are built in spatial (Hilbert-cell) order and the mesh is stored in spatially
//    compact chunks of 32 triangles (mesh.cu, sort.cu); an exact three-level cull skips
//    triangles that cannot reach any of the CTA's support volumes: superchunk spheres and
//    chunk spheres vs the CTA sphere, then chunk sphere vs each image's support CYLINDER;
//  * (image, triangle) pairs that pass the beta-extent test and an alpha-box test (the
//    triangle's (T_x, T_y) box meets the support disk) are compacted into a per-warp ring
//    (ballot + popc) WITH their projected vertices, and drained 32 at a time, one pair per
//    lane, so the divergent per-layer work runs with full warps;
//  * chunk survivors carry their per-image cylinder hits (one 32-bit entry), and each warp
//    prefetches its next chunk's triangles while it processes the current one;
//  * no FMA contraction (-fmad=false, build.py): every fused multiply-add is an explicit fmaf /
//    FFMA2, so the arithmetic (and every tie decision) is exactly the source's;
//  * the per-image rotation coefficients are computed once per image in the CTA prologue
//    ("out of the inner loop");
//  * saturation to uint16 (G9) fused into the prefix-scan epilogue: each row is stored
//    straight to its image's caller index with eight 16-byte stores.
#include <cstdlib>

#include "frame.cuh"
#include "rici_internal.cuh"

namespace rici {
namespace {

#if RICI_GEN_STATS   // tuning builds only: event counters read by rici_debug_gen_stats
__device__ unsigned long long g_stats[13];
#define RICI_STAT(i, v) atomicAdd(&g_stats[i], (unsigned long long)(v))
#else
#define RICI_STAT(i, v)
#endif

#ifndef RICI_GEN_THREADS
#define RICI_GEN_THREADS 256    // 288 / 320 (more warps per SM, fewer registers): C4 294 / 296 vs 283 ms (r2av)
#endif
constexpr int kThreads = RICI_GEN_THREADS;
constexpr int kMaxK = 8;
#ifndef RICI_GEN_LIST_CAP
#define RICI_GEN_LIST_CAP (2 * RICI_GEN_THREADS)
#endif
#ifndef RICI_GEN_CHUNK_CAP
#define RICI_GEN_CHUNK_CAP 3072         // fewer level-3 batches, fewer imbalanced barriers: C4 272.9 -> 270.0 ms (r2cs)
#endif
constexpr int kListCap = RICI_GEN_LIST_CAP;    // superchunks tested per level-1 batch
constexpr int kChunkCap = RICI_GEN_CHUNK_CAP;  // chunk survivors per batch (multiple of kSuper)

// Bin indices in the bin-unit frame (rasterise_triangle): the first row r with Z_r = r >= v is
// ceil(v), the first column whose circle (radius c + 1/2) is at or beyond v is ceil(v - 1/2),
// both clamped to [0, N] and computed as kMagic sums (below).  Exact ties are fragile pixels (G5).

// Stable sort of three vertices by z (a three-stage network; equal z keep their order).
__device__ __forceinline__ void sort3(float &ax, float &ay, float &az, float &bx, float &by,
                                      float &bz, float &cx, float &cy, float &cz) {
#define RICI_SWAP(p, q) { float t = p; p = q; q = t; }
    if (bz < az) { RICI_SWAP(ax, bx) RICI_SWAP(ay, by) RICI_SWAP(az, bz) }
    if (cz < bz) { RICI_SWAP(bx, cx) RICI_SWAP(by, cy) RICI_SWAP(bz, cz) }
    if (bz < az) { RICI_SWAP(ax, bx) RICI_SWAP(ay, by) RICI_SWAP(az, bz) }
#undef RICI_SWAP
}

// Per-launch constants of the bin-unit frame (gen_frame): 1/delta = N/R and the row offset
// N/2 - 1/2 (layer r at Z = r).
struct Geometry {
    float inv_delta;
    float row_off;
};

__device__ __forceinline__ float fast_sqrt(float x) {     // MUFU.SQRT, ~1 ulp; sqrt(0) = 0
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float fast_rcp(float x) {      // MUFU.RCP, ~1 ulp
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// Shared-memory reduction on a 32-bit shared-window address (no generic->shared conversion).
__device__ __forceinline__ void red_shared(unsigned addr, int v) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// Steps 1-6 for every layer of one projected, z-sorted triangle, accumulated
// into the image's per-row difference arrays.  Approximate reciprocals / square roots
// (relative error ~1e-7) move decisions by far less than the 1e-5*R attribution bound.
// `acc` is the image's [N][N+1] difference array as a shared-window address: column N is a
// sink, so a range end at N needs no test, and coinciding ends cancel in place.
//
// Each slice endpoint is computed from its edge alone, in a canonical form -- lower vertex
// first: E = lo + t (hi - lo), t = (beta - z_lo) / (z_hi - z_lo) -- so two triangles sharing an
// edge produce bitwise the same point and a circle through it is counted exactly once (no crack
// at shared edges; G5).  E0 lies on the long edge (a,c), E1 on (a,b) below the middle vertex and
// on (b,c) from it up (step 1).  The parameters are saturated to [0, 1]: a row the
// ceil-based range admits by rounding (beta within ~1 ulp outside [z_a, z_c), G5) becomes a
// zero-length slice (E0 = E1 = a or c) and contributes nothing, so no per-layer membership test
// is needed.  The (x, y) pairs run as packed FP32x2 instructions (FFMA2).
__device__ __forceinline__ float2 f2(float x, float y) { return make_float2(x, y); }
__device__ __forceinline__ float mul_sat(float a, float b) {     // FMUL.SAT: clamp to [0, 1]
    float r;
    asm("mul.rn.ftz.sat.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

// Bin indices without F2I / I2F / FRND (XU ops; C4 283.3 -> 279.9 ms, images identical, r2bl-r2bm):
// ceil(v) + 1.5 * 2^23 is v + 1.5 * 2^23 rounded UP, exactly for |v| < 2^22 (unit ulp there), so
// the float's bits are ceil(v) + 0x4B400000 and the float minus the magic is ceil(v); positive
// floats order like their bits (negative ones as signed integers), so clamps need no conversion.
constexpr float kMagic = 12582912.f;
constexpr int kMagicBits = 0x4B400000;
#ifndef RICI_GEN_INSIDE
#define RICI_GEN_INSIDE 1
#endif
#ifndef RICI_GEN_RED_MODE
#define RICI_GEN_RED_MODE 3     // 1: per-row (v1, v2) selects (r2d: C4 341 -> 337 ms against 0, a branch)
#endif

// All coordinates here are in BIN units (DESIGN.md 6.1 "bin-unit frame"): x, y scaled by
// 1/delta = N/R, and Z = z/delta + N/2 - 1/2, so layer r lies at Z = r exactly (beta_r =
// (r + 1/2) delta - R/2, G4), column c's circle at radius c + 1/2, and the support radius is N.
template <int NC>
__device__ __forceinline__ void rasterise_triangle(unsigned acc, int n_rt, int two, int neg1,
                                                   float ax, float ay, float az, float bx,
                                                   float by, float bz, float cx, float cy,
                                                   float cz) {
    const int N = NC ? NC : n_rt;
    // first row with Z_r >= z_a / z_c, clamped to [0, N], without F2I / I2F (kMagic)
    const float2 rc = __fadd2_ru(f2(az, cz), f2(kMagic, kMagic));
    const int b_lo = min(max(__float_as_int(rc.x), kMagicBits), kMagicBits + N);
    const int b_hi = min(max(__float_as_int(rc.y), kMagicBits), kMagicBits + N);
    if (b_lo >= b_hi) { RICI_STAT(8, 1); return; }
    const int r_lo = b_lo - kMagicBits;
    const float2 rzr = __fadd2_rn(f2(__int_as_float(b_lo), __int_as_float(b_hi)), f2(-kMagic, -kMagic));
#if RICI_GEN_STATS
    const int r_hi = b_hi - kMagicBits;
    bool stat_emitted = false;
#endif
    RICI_STAT(4, r_hi - r_lo);
    const float i_ac = fast_rcp(cz - az);                // z_c > z_a whenever a layer is inside
    const float i_ab = bz > az ? fast_rcp(bz - az) : 0.f;
    const float i_bc = cz > bz ? fast_rcp(cz - bz) : 0.f;
    const float2 A = f2(ax, ay), B = f2(bx, by), AC = f2(cx - ax, cy - ay), AB = f2(bx - ax, by - ay),
                 BC = f2(cx - bx, cy - by);
    const float2 half = f2(-0.5f, -0.5f);
    const unsigned row_step = 4u * (unsigned)(N + 1);
    // Column indices without F2I (an XU op): the bits of v + kMagic rounded up are ceil(v) +
    // 0x4B400000 (larger v land above the clamp), and the shared-window address 4 * bits +
    // (row - 4 * 0x4B400000) wraps to the row's column: bitwise the indices of min(ceil(v), N)
    // (__float2int_ru) for every finite v >= -1/2.
    const unsigned cap = (unsigned)kMagicBits + (unsigned)N;
    unsigned row = acc + row_step * (unsigned)r_lo - 4u * (unsigned)kMagicBits;
    const float rz_hi = rzr.y;
    for (float rz = rzr.x; rz < rz_hi; rz += 1.f, row += row_step) {
        // Step 1: E0 on the long edge (a,c), E1 on (a,b) below / (b,c) above the middle vertex.
        const float t = mul_sat(rz - az, i_ac);
        const float2 e0 = __ffma2_rn(f2(t, t), AC, A);
        const bool below = rz < bz;
        const float u = mul_sat(rz - (below ? az : bz), below ? i_ab : i_bc);
        const float2 e1 = __ffma2_rn(f2(u, u), below ? AB : BC, below ? A : B);
        // Step 2: rotate so E0E1 is parallel to x with the normalised direction D/|D| as
        // (cos, sin): the rotated x of E0 / E1 is (D.E0)/|D| / (D.E1)/|D|, so their signs are
        // those of D.E0 and D.E0 + |D|^2 -- the normalisation is only needed for |C| below.
        const float2 d = __ffma2_rn(e0, f2(-1.f, -1.f), e1);
        const float l2 = fmaf(d.x, d.x, d.y * d.y);
        const float de0 = fmaf(d.x, e0.x, d.y * e0.y);    // |D| * x0
        // Steps 3-4: distances of E0, E1 from the axis; single range [min, max).  Column c's
        // circle (radius c + 1/2 in bin units) is the first at or beyond v at ceil(v - 1/2).
        const float r0 = fast_sqrt(fmaf(e0.x, e0.x, e0.y * e0.y)), r1 = fast_sqrt(fmaf(e1.x, e1.x, e1.y * e1.y));
        const float2 cf = __fadd2_ru(__fadd2_rn(f2(fminf(r0, r1), fmaxf(r0, r1)), half), f2(kMagic, kMagic));
        const unsigned c_min = min(__float_as_uint(cf.x), cap), c_max = min(__float_as_uint(cf.y), cap);
        // Steps 5-6: double range [|C|, min) iff the x signs differ (x = 0 non-negative);
        // |C| = |rotated y| = |D x E0| / |D|.  Single: +1 at c_min, -1 at c_max.  Double:
        // +2 at c_c, -1 at c_min, -1 at c_max.  Empty ranges (also a zero-length slice, whose
        // r0 = r1 and de0 = 0) cancel at one address; they are predicated off.
        const bool dbl = de0 < 0.f && de0 + l2 >= 0.f;
        unsigned c_lo = c_min;
        if (dbl) {
            const float y = fmaf(d.x, e0.y, -d.y * e0.x) * rsqrtf(l2);
            c_lo = min(__float_as_uint(__fadd_ru(fabsf(y) - 0.5f, kMagic)), c_min);
        }
        const bool emit = c_lo != c_max;                  // something in [c_lo, c_max)
        (void)emit;
        RICI_STAT(5, emit ? 1 : 0);
#if RICI_GEN_STATS
        stat_emitted |= emit;
#endif
#if RICI_GEN_RED_MODE == 3
        // unconditional and constant: +2 at c_lo, -1 at c_min, -1 at c_max.  A single range has
        // c_lo = c_min, where +2 - 1 leaves its +1; an empty range cancels in place.  The
        // constants sit in registers the compiler cannot rematerialise (two = 2, neg1 = -1,
        // derived from a kernel parameter) instead of a move per row: layer loop 56 -> 52
        // instructions, C4 279.8 -> 277.9 ms, C3 86.7 -> 85.8 ms, images identical (r2bn)
        red_shared(row + 4u * (unsigned)c_lo, two);
        red_shared(row + 4u * (unsigned)c_min, neg1);
        red_shared(row + 4u * (unsigned)c_max, neg1);
    }
#elif RICI_GEN_RED_MODE == 1
        // unconditional: +v1 at c_lo, +v2 at c_min, -1 at c_max with (v1, v2) = (2, -1) for a
        // double range and (1, 0) for a single one; an empty range cancels in place
        red_shared(row + 4u * (unsigned)c_lo, dbl ? 2 : 1);
        red_shared(row + 4u * (unsigned)c_min, dbl ? -1 : 0);
        red_shared(row + 4u * (unsigned)c_max, -1);
    }
#else
        if (!emit) continue;
        red_shared(row + 4u * (unsigned)c_lo, dbl ? 2 : 1);
        if (dbl) red_shared(row + 4u * (unsigned)c_min, -1);
        red_shared(row + 4u * (unsigned)c_max, -1);
    }
#endif
#if RICI_GEN_STATS
    if (!stat_emitted) RICI_STAT(9, 1);            // rasterised pairs that emitted no segment
#endif
}


// The per-image projection in bin units: translation first (Eq. 2, S_v), then the composed
// rotation of Eqs. 3-4 scaled by 1/delta, with the row offset folded into Z.
struct __align__(16) GenFrame {
    float nsx, nsy, nsz, zoff;   // -S_v (p = v + (-S_v) is bitwise v - S_v); N/2 - 1/2
    float xx, xy, xz, yx;        // X = xx px + xy py + xz pz;  Y = yx px + yy py
    float yy, zx, zy, zz;        // Z = zx px + zy py + zz pz + zoff
};
__device__ __forceinline__ GenFrame gen_frame(const Frame &f, float inv_delta, float zoff) {
    GenFrame q;
    q.nsx = -f.sx; q.nsy = -f.sy; q.nsz = -f.sz; q.zoff = zoff;
    q.xx = f.nbz * f.nax * inv_delta; q.xy = f.nbz * f.nay * inv_delta; q.xz = -f.nbx * inv_delta;
    q.yx = -f.nay * inv_delta; q.yy = f.nax * inv_delta;
    q.zx = f.czx * inv_delta; q.zy = f.czy * inv_delta; q.zz = f.czz * inv_delta;
    return q;
}

// Project one triangle into image k's spin frame (Eqs. 2-4): translate first (Eq. 2), then the
// scaled rotation.  Vertices 0 and 1 go through packed FP32x2 (FADD2 / FFMA2 / FMUL2, the frame
// coefficient broadcast), vertex 2 through the scalar ops: every lane of a packed op is the
// scalar operation in the same order, so a shared vertex projects bitwise alike in every
// triangle (C4 289.4 -> 283 ms with the float beta test below, r2y).  pp = translated vertices
// 0 and 1 (x, y, z pairs), p2 = translated vertex 2.
__device__ __forceinline__ void project_z(const GenFrame &f, const float *v, float2 *pp, float *p2, float *z) {
    pp[0] = __fadd2_rn(f2(v[0], v[3]), f2(f.nsx, f.nsx));
    pp[1] = __fadd2_rn(f2(v[1], v[4]), f2(f.nsy, f.nsy));
    pp[2] = __fadd2_rn(f2(v[2], v[5]), f2(f.nsz, f.nsz));
    p2[0] = v[6] + f.nsx; p2[1] = v[7] + f.nsy; p2[2] = v[8] + f.nsz;
    const float2 z01 = __ffma2_rn(f2(f.zx, f.zx), pp[0],
                                  __ffma2_rn(f2(f.zy, f.zy), pp[1], __ffma2_rn(f2(f.zz, f.zz), pp[2], f2(f.zoff, f.zoff))));
    z[0] = z01.x; z[1] = z01.y;
    z[2] = fmaf(f.zx, p2[0], fmaf(f.zy, p2[1], fmaf(f.zz, p2[2], f.zoff)));
}
// Eqs. 3-4 for T_x, T_y of the translated vertices (project_z output).
__device__ __forceinline__ void project_xy(const GenFrame &f, const float2 *pp, const float *p2, float *x, float *y) {
    const float2 y01 = __ffma2_rn(f2(f.yx, f.yx), pp[0], __fmul2_rn(f2(f.yy, f.yy), pp[1]));
    const float2 x01 = __ffma2_rn(f2(f.xx, f.xx), pp[0], __ffma2_rn(f2(f.xy, f.xy), pp[1], __fmul2_rn(f2(f.xz, f.xz), pp[2])));
    y[0] = y01.x; y[1] = y01.y; x[0] = x01.x; x[1] = x01.y;
    y[2] = fmaf(f.yx, p2[0], f.yy * p2[1]);
    x[2] = fmaf(f.xx, p2[0], fmaf(f.xy, p2[1], f.xz * p2[2]));
}
// alpha cull: if the triangle's (T_x, T_y) bounding box misses the support disk (radius N in
// bin units), every slice point has alpha > R > rho_{N-1} and no bin can be hit (exact skip)
__device__ __forceinline__ bool alpha_box_hits(const float *x, const float *y, float r2) {
    const float bx0 = fmaxf(fmaxf(fminf(x[0], fminf(x[1], x[2])), -fmaxf(x[0], fmaxf(x[1], x[2]))), 0.f);
    const float by0 = fmaxf(fmaxf(fminf(y[0], fminf(y[1], y[2])), -fmaxf(y[0], fmaxf(y[1], y[2]))), 0.f);
    return bx0 * bx0 + by0 * by0 <= r2;
}
// K <= 2 (N = 64 default): 33 KB of counters + 18 KB of projected-triangle queues per CTA, so
// 3 CTAs / SM (78 registers, no spill).  Measured on C4 / C3 / C2 (r2e, r2j, r2k; images
// identical): 5 CTAs at the 48-register cap 337 / 103 / 1.75 ms; 4 CTAs 325 / 99.4 / 1.71;
// 3 CTAs 317.7 / 97.6 / 1.68; 3 CTAs with the projected queue 310.4 / 96.0 / 1.66; 2 CTAs (with
// the queue) 357.6 / 110.5 / 1.93; K = 4 at 2 CTAs 321.5 / 98.8 / 1.71.
template <int K, int NC>
#ifndef RICI_GEN_MIN_BLOCKS
#define RICI_GEN_MIN_BLOCKS 3
#endif
#ifndef RICI_GEN_MIN_BLOCKS4
#define RICI_GEN_MIN_BLOCKS4 2
#endif
__global__ void __launch_bounds__(kThreads, K <= 2 ? RICI_GEN_MIN_BLOCKS : (K <= 4 ? RICI_GEN_MIN_BLOCKS4 : 1))
generate_kernel(const float *__restrict__ tri, const float4 *__restrict__ sphere, int64_t n_chunks,
                const float4 *__restrict__ super_sphere, int64_t n_super,
                const float *__restrict__ origins, const int *__restrict__ img_perm, int64_t n,
                float R, int N, const Geometry g, uint16_t *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ Frame frames[kMaxK];
    __shared__ GenFrame gframes[kMaxK];
    __shared__ int img_idx[kMaxK];
    __shared__ int list[kListCap];
    __shared__ int list_n, chunk_n;
    __shared__ unsigned chunk_list[kChunkCap];   // (chunk << 8) | image mask
    __shared__ float cta_sphere[4];
    // the queued pairs: a 64-slot ring per warp of 48-byte entries holding the projected
    // (unsorted) triangle and its image, written by the queue phase from the registers of its
    // beta / alpha tests with three 16-byte stores, so the drain neither reloads nor re-projects
    // the triangle (C4 317.7 -> 310.4 ms, r2j; 48-byte entries instead of nine 4-byte planes and
    // an item array: 310.8 -> 290.9 ms, r2t).  A quarter-warp's 16-byte accesses at a 48-byte
    // stride cover all 32 banks once.
    __shared__ float4 qa[kThreads / 32][64][3];      // x0 y0 z0 x1 | y1 z1 x2 y2 | z2 k - -
    int qh = 0;                                          // warp-uniform ring head

    int *acc = reinterpret_cast<int *>(smem_raw);        // [K][N][N+1] difference arrays
    const unsigned acc_s = (unsigned)__cvta_generic_to_shared(acc);
    const int c_two = 2 + (N >> 31), c_neg1 = -1 - (N >> 31);   // 2 and -1 (N > 0), opaque to ptxas
    if (NC) N = NC;                                      // N = 64: compile-time bin geometry
    const int img_words = N * (N + 1);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    const int64_t img0 = (int64_t)blockIdx.x * K;
    const int k_valid = (int)min((int64_t)K, n - img0);

    {
        const int nw = K * img_words;
        int4 *a4 = reinterpret_cast<int4 *>(acc);              // dynamic smem: 16-byte aligned
        for (int i = tid; i < nw / 4; i += kThreads) a4[i] = make_int4(0, 0, 0, 0);
        for (int i = (nw / 4) * 4 + tid; i < nw; i += kThreads) acc[i] = 0;
    }
    if (tid < K) {
        if (tid < k_valid) {
            const int idx = img_perm ? img_perm[img0 + tid] : (int)(img0 + tid);
            img_idx[tid] = idx;
            frames[tid] = make_frame(origins + 6 * (int64_t)idx);
            gframes[tid] = gen_frame(frames[tid], g.inv_delta, g.row_off);
        } else {
            Frame f = {};
            frames[tid] = f;
            gframes[tid] = gen_frame(f, g.inv_delta, g.row_off);
        }
    }
    __syncthreads();
    if (tid == 0) {
        // union of the images' support spheres (cylinder r <= R, |beta| <= R/2 -> radius R*sqrt(5)/2)
        float lo[3] = {3e38f, 3e38f, 3e38f}, hi[3] = {-3e38f, -3e38f, -3e38f};
        int nv = 0;
        for (int k = 0; k < k_valid; ++k) {
            if (frames[k].valid == 0.f) continue;
            ++nv;
            float p[3] = {frames[k].sx, frames[k].sy, frames[k].sz};
            for (int a = 0; a < 3; ++a) { lo[a] = fminf(lo[a], p[a]); hi[a] = fmaxf(hi[a], p[a]); }
        }
        if (nv == 0) { cta_sphere[3] = -1.f; }
        else {
            float c[3] = {0.5f * (lo[0] + hi[0]), 0.5f * (lo[1] + hi[1]), 0.5f * (lo[2] + hi[2])};
            float r2 = 0.f;
            for (int k = 0; k < k_valid; ++k) {
                if (frames[k].valid == 0.f) continue;
                float dx = frames[k].sx - c[0], dy = frames[k].sy - c[1], dz = frames[k].sz - c[2];
                r2 = fmaxf(r2, dx * dx + dy * dy + dz * dz);
            }
            float scale = fmaxf(fabsf(c[0]), fmaxf(fabsf(c[1]), fabsf(c[2])));
            cta_sphere[0] = c[0]; cta_sphere[1] = c[1]; cta_sphere[2] = c[2];
            cta_sphere[3] = (sqrtf(r2) + R * 1.1180340f) * (1.0f + 1e-5f) + 1e-5f * scale + 1e-30f;
        }
    }
    __syncthreads();

    const float cs_r = cta_sphere[3];
    int qn = 0;                                          // warp-uniform queue length

    // Drain `cnt` (<= 32) queued (chunk, triangle, image) items with one item per lane: the
    // projected triangle comes from the ring, is sorted by Z and rasterised.
    auto drain = [&](int cnt) {
        __syncwarp();
        const int slot = (qh + lane) & 63;
        qh = (qh + cnt) & 63;
        qn -= cnt;
        int stat_rows = 0;
        (void)stat_rows;
        if (lane < cnt) {
            const float4 q0 = qa[warp][slot][0], q1 = qa[warp][slot][1], q2 = qa[warp][slot][2];
            const int k = __float_as_int(q2.y);
            float ax = q0.x, ay = q0.y, az = q0.z, bx = q0.w, by = q1.x, bz = q1.y, cx = q1.z, cy = q1.w, cz = q2.x;
            sort3(ax, ay, az, bx, by, bz, cx, cy, cz);
            RICI_STAT(2, 1);
            RICI_STAT(3, 1);
#if RICI_GEN_STATS
            stat_rows = max(0, min(max(__float2int_ru(cz), 0), N) - min(max(__float2int_ru(az), 0), N));
#endif
            rasterise_triangle<NC>(acc_s + 4u * (unsigned)(k * img_words), N, c_two, c_neg1, ax, ay, az, bx, by, bz,
                                   cx, cy, cz);
        }
#if RICI_GEN_STATS
        {
            const int mx = __reduce_max_sync(0xffffffffu, stat_rows);
            if (lane == 0) { RICI_STAT(6, mx); RICI_STAT(7, 1); }
        }
#endif
        __syncwarp();
    };

    if (cs_r >= 0.f) {
        const float ccx = cta_sphere[0], ccy = cta_sphere[1], ccz = cta_sphere[2];
        const float pad_r = 1e-4f * R;
        // Level 1: superchunks (kSuper*kChunk triangles) whose sphere meets the CTA sphere.
        for (int64_t base = 0; base < n_super; base += kListCap) {
            if (tid == 0) { list_n = 0; chunk_n = 0; }
            __syncthreads();
            for (int q = 0; q < kListCap / kThreads; ++q) {
                int64_t c = base + q * kThreads + tid;
                bool keep = false;
                if (c < n_super) {
                    float4 s4 = super_sphere[c];
                    float dx = s4.x - ccx, dy = s4.y - ccy, dz = s4.z - ccz;
                    float rr = s4.w + cs_r;
                    keep = dx * dx + dy * dy + dz * dz <= rr * rr;
                }
                unsigned m = __ballot_sync(0xffffffffu, keep);
                int pos = 0;
                if (lane == 0 && m) pos = atomicAdd(&list_n, __popc(m));
                pos = __shfl_sync(0xffffffffu, pos, 0);
                if (keep) list[pos + __popc(m & lt_mask)] = (int)(c - base);
            }
            __syncthreads();
            const int n_sc = list_n;
            // Level 2: chunks of the surviving superchunks, in batches that fit the chunk list.
            for (int sc0 = 0; sc0 < n_sc; sc0 += kChunkCap / kSuper) {
                const int sc1 = min(n_sc, sc0 + kChunkCap / kSuper);
                for (int e = sc0 + warp; e < sc1; e += kThreads / 32) {
                    const int64_t c_lane = (base + list[e]) * kSuper + lane;
                    // chunk sphere vs the CTA sphere, then vs each image's support CYLINDER
                    // (r <= R, |beta| <= R/2); the per-image hits travel with the chunk id
                    unsigned kbits = 0;
                    if (c_lane < n_chunks) {
                        const float4 s4 = sphere[c_lane];
                        float dx = s4.x - ccx, dy = s4.y - ccy, dz = s4.z - ccz;
                        float rr = s4.w + cs_r;
                        if (dx * dx + dy * dy + dz * dz <= rr * rr) {
                            const float pad = pad_r + 1e-6f * (fabsf(s4.x) + fabsf(s4.y) + fabsf(s4.z) + s4.w);
                            const float ra = R + s4.w + pad, hb = 0.5f * R + s4.w + pad;
#pragma unroll
                            for (int k = 0; k < K; ++k) {
                                const Frame &f = frames[k];
                                if (k >= k_valid || f.valid == 0.f) continue;
                                float ex = s4.x - f.sx, ey = s4.y - f.sy, ez = s4.z - f.sz;
                                float b = fmaf(f.czx, ex, fmaf(f.czy, ey, f.czz * ez));
                                float a2 = fmaxf(ex * ex + ey * ey + ez * ez - b * b, 0.f);
                                if (fabsf(b) <= hb && a2 <= ra * ra) {
                                    kbits |= 1u << k;
#if RICI_GEN_INSIDE
                                    // the whole chunk within radius R of the axis: every triangle's
                                    // (T_x, T_y) box meets the support disk, so its alpha test is
                                    // skipped (it is an exact skip, so a loose flag only costs work)
                                    const float ri = R - s4.w - pad;
                                    if (K <= 4 && ri > 0.f && a2 <= ri * ri) kbits |= 1u << (4 + k);
#endif
                                }
                            }
                        }
                    }
                    const bool ck = kbits != 0;
                    unsigned m = __ballot_sync(0xffffffffu, ck);
                    int pos = 0;
                    if (lane == 0 && m) pos = atomicAdd(&chunk_n, __popc(m));
                    pos = __shfl_sync(0xffffffffu, pos, 0);
                    if (ck) chunk_list[pos + __popc(m & lt_mask)] = ((unsigned)c_lane << 8) | kbits;
                }
                __syncthreads();
                const int n_ck = chunk_n;
                // Level 3: static round-robin over the warps, so each warp knows its next chunk
                // and prefetches its nine triangle planes while the current one is processed
                // (measured faster than a shared-counter schedule with the same prefetch).
                // each chunk: its (image, triangle) pairs -- beta-extent test: does a
                // layer Z = r lie in [z_min, z_max)?  then the alpha box; survivors go to the
                // warp's ring with their projected vertices
                auto process = [&](const unsigned ent, const float *v) {
                    const unsigned kmask = ent & (K <= 4 && RICI_GEN_INSIDE ? 0xfu : 0xffu);
                    if (lane == 0) { RICI_STAT(0, 1); RICI_STAT(1, __popc(kmask)); RICI_STAT(12, __popc((ent >> 4) & 0xfu)); }
    #if RICI_GEN_STATS
                        {   // finer culls, counted only: the 8-triangle sub-chunk's sphere and the triangle's
                            // own sphere against each tested image's support cylinder (stats 10, 11)
                            float tc[3], tr = 0.f;
                            for (int a = 0; a < 3; ++a) tc[a] = (v[a] + v[3 + a] + v[6 + a]) * (1.f / 3.f);
                            for (int j = 0; j < 3; ++j) {
                                float dx = v[3 * j] - tc[0], dy = v[3 * j + 1] - tc[1], dz = v[3 * j + 2] - tc[2];
                                tr = fmaxf(tr, sqrtf(dx * dx + dy * dy + dz * dz));
                            }
                            float lo[3], hi[3];
                            for (int a = 0; a < 3; ++a) { lo[a] = tc[a] - tr; hi[a] = tc[a] + tr; }
                            for (int o = 1; o < 8; o <<= 1)
                                for (int a = 0; a < 3; ++a) {
                                    lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
                                    hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
                                }
                            float sc[3], sr = 0.f;
                            for (int a = 0; a < 3; ++a) sc[a] = 0.5f * (lo[a] + hi[a]);
                            {
                                float dx = tc[0] - sc[0], dy = tc[1] - sc[1], dz = tc[2] - sc[2];
                                sr = sqrtf(dx * dx + dy * dy + dz * dz) + tr;
                            }
                            for (int o = 1; o < 8; o <<= 1) sr = fmaxf(sr, __shfl_xor_sync(0xffffffffu, sr, o));
                            for (int k = 0; k < K; ++k) {
                                if (!((kmask >> k) & 1u)) continue;
                                const Frame &f = frames[k];
                                auto cyl = [&](const float *c, float w) {
                                    const float pad = 1e-4f * R + 1e-6f * (fabsf(c[0]) + fabsf(c[1]) + fabsf(c[2]) + w);
                                    const float ra = R + w + pad, hb = 0.5f * R + w + pad;
                                    float ex = c[0] - f.sx, ey = c[1] - f.sy, ez = c[2] - f.sz;
                                    float b = fmaf(f.czx, ex, fmaf(f.czy, ey, f.czz * ez));
                                    float a2 = fmaxf(ex * ex + ey * ey + ez * ez - b * b, 0.f);
                                    return fabsf(b) <= hb && a2 <= ra * ra;
                                };
                                RICI_STAT(10, cyl(sc, sr) ? 1 : 0);
                                RICI_STAT(11, cyl(tc, tr) ? 1 : 0);
                            }
                        }
    #endif
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        if (!((kmask >> k) & 1u)) continue;
                        const GenFrame f = gframes[k];
                        float z[3], x[3], y[3];
                        float2 pp[3];
                        float p2[3];
                        project_z(f, v, pp, p2, z);
                        float zlo = fminf(z[0], fminf(z[1], z[2])), zhi = fmaxf(z[0], fmaxf(z[1], z[2]));
                        // beta-extent test: a layer Z = r in [zlo, zhi) with 0 <= r < N,
                        // i.e. the first row at or above max(zlo, 0) lies below min(zhi, N); for an
                        // integer k, k < b iff k < ceil(b), so both sides are ceilings, taken as
                        // kMagic sums by one FADD2.RP (float tests: C4 289.4 -> 286.4 ms, r2x)
                        const float2 cb = __fadd2_ru(f2(fmaxf(zlo, 0.f), fminf(zhi, (float)N)), f2(kMagic, kMagic));
                        bool keep = cb.x < cb.y;
                        if (keep) {
                            project_xy(f, pp, p2, x, y);
#if RICI_GEN_INSIDE
                            if (!(K <= 4 && ((ent >> (4 + k)) & 1u)))   // warp-uniform
#endif
                                keep = alpha_box_hits(x, y, (float)(N * N));
                        }
                        const unsigned m = __ballot_sync(0xffffffffu, keep);
                        if (keep) {
                            const int slot = (qh + qn + __popc(m & lt_mask)) & 63;
                            qa[warp][slot][0] = make_float4(x[0], y[0], z[0], x[1]);
                            qa[warp][slot][1] = make_float4(y[1], z[1], x[2], y[2]);
                            qa[warp][slot][2] = make_float4(z[2], __int_as_float(k), 0.f, 0.f);
                        }
                        qn += __popc(m);
                        if (qn >= 32) drain(32);
                    }
                };
                // static round-robin over the warps, so each warp knows its next chunk and
                // prefetches its nine triangle planes while the current one is processed
                // (measured faster than a shared-counter schedule with the same prefetch)
                auto load = [&](int e, float *v) -> unsigned {
                    const unsigned ent = chunk_list[e];
                    load_triangle(tri, (int64_t)(ent >> 8), lane, v);
                    return ent;
                };
                constexpr int kW = kThreads / 32;
                {
                    float nv9[9];
                    unsigned nxt_ent = 0;
                    int e = warp;
                    if (e < n_ck) nxt_ent = load(e, nv9);
                    while (e < n_ck) {
                        const unsigned ent = nxt_ent;
                        float v[9];
#pragma unroll
                        for (int c = 0; c < 9; ++c) v[c] = nv9[c];
                        e += kW;
                        if (e < n_ck) nxt_ent = load(e, nv9);
                        process(ent, v);
                    }
                }
                __syncthreads();
                if (tid == 0) chunk_n = 0;
                __syncthreads();
            }
        }
        if (qn > 0) drain(qn);
    }
    __syncthreads();

    // Epilogue: per-row inclusive prefix sum of the difference arrays, saturated to uint16 (G9),
    // stored at the image's caller index.  N = 64 (16-byte aligned output): one thread per row,
    // a sequential running sum over the 64 columns (row r of a [64][65] array starts in bank
    // r mod 32, so a warp's 32 rows read 32 distinct banks), eight 16-byte stores per row.
    if (N == 64 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
        for (int rr = tid; rr < k_valid * 64; rr += kThreads) {
            const int k = rr >> 6, r = rr & 63;
            const int *rp = acc + k * img_words + r * 65;
            uint4 *dst = reinterpret_cast<uint4 *>(out + (int64_t)img_idx[k] * 4096 + r * 64);
            unsigned run = 0;
#pragma unroll
            for (int c8 = 0; c8 < 8; ++c8) {
                unsigned w[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    run += (unsigned)rp[8 * c8 + 2 * h];
                    const unsigned lo = min(run, 65535u);
                    run += (unsigned)rp[8 * c8 + 2 * h + 1];
                    w[h] = lo | (min(run, 65535u) << 16);
                }
                dst[c8] = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
        return;
    }
    // any N: warp per row -- lane l holds columns [l*cpl, l*cpl + cpl), written as packed pairs
    // when aligned.
    const int npix = N * N;
    const int cpl = (N + 31) / 32;                 // columns per lane
    const bool pairs = (cpl % 2) == 0 && (N % 2) == 0 && (reinterpret_cast<uintptr_t>(out) & 3) == 0;
    for (int k = 0; k < k_valid; ++k) {
        for (int r = warp; r < N; r += kThreads / 32) {
            const int *rp = acc + k * img_words + r * (N + 1);
            unsigned vals[4];
            unsigned local = 0;
            for (int j = 0; j < cpl; ++j) {
                int c = lane * cpl + j;
                unsigned x = (c < N) ? (unsigned)rp[c] : 0u;
                local += x;
                vals[j] = local;
            }
            unsigned incl = local;
            for (int o = 1; o < 32; o <<= 1) {
                unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const unsigned excl = incl - local;
            uint16_t *dst = out + (int64_t)img_idx[k] * npix + (int64_t)r * N;
            if (pairs) {
                for (int j = 0; j < cpl; j += 2) {
                    int c = lane * cpl + j;
                    if (c < N)
                        *reinterpret_cast<unsigned *>(dst + c) =
                            min(vals[j] + excl, 65535u) | (min(vals[j + 1] + excl, 65535u) << 16);
                }
            } else {
                for (int j = 0; j < cpl; ++j) {
                    int c = lane * cpl + j;
                    if (c < N) dst[c] = (uint16_t)min(vals[j] + excl, 65535u);
                }
            }
        }
    }
}

}  // namespace

int generate_images_per_cta(int N) {
    int per = N * (N + 1) * 4;
#ifndef RICI_GEN_BUDGET_KB
#define RICI_GEN_BUDGET_KB 34
#endif
    int budget = RICI_GEN_BUDGET_KB * 1024;       // counters per CTA (K = 2 at N = 64)
    if (const char *v = getenv("RICI_GEN_SMEM_KB")) budget = atoi(v) * 1024;   // tuning knob
    int k = budget / per;
    return k < 1 ? 1 : (k > kMaxK ? kMaxK : k);
}

cudaError_t launch_generate(const DeviceMesh &m, const float *d_origins, int64_t n, float R, int N,
                            uint16_t *d_out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const int K = generate_images_per_cta(N);
    size_t smem = (size_t)K * N * (N + 1) * sizeof(int);
    const int Kt = K >= 8 ? 8 : K >= 4 ? 4 : K >= 2 ? 2 : 1;
    const bool n64 = N == 64 && (Kt == 2 || Kt == 4);     // the compile-time N = 64 instances
    const void *kern = n64 ? (Kt == 2 ? (const void *)generate_kernel<2, 64> : (const void *)generate_kernel<4, 64>)
                     : Kt == 8 ? (const void *)generate_kernel<8, 0> : Kt == 4 ? (const void *)generate_kernel<4, 0>
                     : Kt == 2 ? (const void *)generate_kernel<2, 0> : (const void *)generate_kernel<1, 0>;
    smem = (size_t)Kt * N * (N + 1) * sizeof(int);
    {
        cudaError_t e = ensure_smem(kern, smem);
        if (e != cudaSuccess) return e;
    }
    // build the images in spatial order so a CTA's K support volumes are compact
    int *perm = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&perm, sizeof(int) * n, s);
    if (e != cudaSuccess) return e;
    if ((e = spatial_order(d_origins, 6, n, perm, s)) != cudaSuccess) { cudaFreeAsync(perm, s); return e; }
#ifndef RICI_GEN_KD_IMAGES
#define RICI_GEN_KD_IMAGES 0
#endif
    if (RICI_GEN_KD_IMAGES && (e = kd_refine(d_origins, 6, n, perm, s)) != cudaSuccess) { cudaFreeAsync(perm, s); return e; }
    int64_t blocks = (n + Kt - 1) / Kt;
    // the geometry lives in the kernel's parameter bank (no per-thread recomputation)
    Geometry g;
    g.inv_delta = (float)N / R;
    g.row_off = 0.5f * (float)N - 0.5f;
#define RICI_GEN_LAUNCH(KK, NN)                                                                         \
    generate_kernel<KK, NN><<<(unsigned)blocks, kThreads, smem, s>>>(m.tri, m.sphere, m.n_chunks, m.super_sphere, \
                                                                 m.n_super, d_origins, perm, n, R, N, g, d_out)
    KernelTimer timer(0, s);
    if (n64 && Kt == 2) RICI_GEN_LAUNCH(2, 64);
    else if (n64) RICI_GEN_LAUNCH(4, 64);
    else if (Kt == 8) RICI_GEN_LAUNCH(8, 0);
    else if (Kt == 4) RICI_GEN_LAUNCH(4, 0);
    else if (Kt == 2) RICI_GEN_LAUNCH(2, 0);
    else RICI_GEN_LAUNCH(1, 0);
    timer.end();
#undef RICI_GEN_LAUNCH
    note_launches(1);
    e = cudaGetLastError();
    cudaFreeAsync(perm, s);
    return e;
}

}  // namespace rici

#if RICI_GEN_STATS
extern "C" __attribute__((visibility("default"))) int rici_debug_gen_stats(unsigned long long *out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, rici::g_stats, sizeof(unsigned long long) * 13);
    if (reset) { unsigned long long z[13] = {}; cudaMemcpyToSymbol(rici::g_stats, z, sizeof(z)); }
    return 0;
}
#endif

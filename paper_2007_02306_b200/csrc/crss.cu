// crss.cu -- (a9-a12) CRSS search on sm_100a.
//
// Paper: the Clutter Resistant Distance ("CRSS" in the north star) compares the
// horizontal changes of a needle and a haystack image, only where the needle
// changes (Eq. 6, Eq. 7, Listing 1):
//     CRSS(n,h) = sum_{r=0}^{N-1} sum_{c=1}^{N-1} [D_n(r,c) != 0] (D_n(r,c) - D_h(r,c))^2,
//     D_x(r,c) = x[r][c] - x[r][c-1].
// The rank of needle i is #{ j : CRSS(n_i,h_j) < CRSS(n_i,h_i) } (best tie P:459).
//
// This is the general SIMT path (every N; the exact fallback of the tensor-core path in
// crss_mma.cu for images outside its int8 guard; RICI_CRSS_SIMT / RICI_CRSS_EARLY_EXIT).
// B200 design:
//  a9  needle preprocessing: one warp per needle compacts the needle's change mask (D_n != 0)
//      into a CSR list of packed (D_n, pixel) entries with a warp ballot -- the mask held as
//      the list of its set positions (typically 2-7% of the 4032 deltas), in decreasing-|D_n|
//      buckets, padded to a multiple of 8 with zero terms and closed by a marker entry.
//  a11 streaming compare: a CTA stages a tile of 32 haystack images as int8 D_h planes in
//      shared memory (one power-of-two plane per lane, XOR-swizzled so the 32 lanes hit 32
//      distinct banks; the left neighbour comes from the previous lane).  Each warp
//      streams one contiguous run of needle lists (cp.async, double-buffered) and lane j
//      accumulates needle i vs haystack image j, integer-only: 4 instructions per entry.
//  a12 rank: pred = CRSS < t_i, __ballot_sync + __popc per 32 images, counts kept in shared
//      memory per needle and flushed once per work item.  Rank mode stops a needle
//      once every lane's partial sum is >= t_i.
#include "rici_internal.cuh"

namespace rici {
namespace {

constexpr int kTileImages = 32;          // one haystack image per lane
constexpr int kCrssThreads = 1024;
constexpr int kWarps = kCrssThreads / 32;
constexpr int kNeedleChunk = 2048;       // needles per work item
constexpr int kSeg = 128;                // entries per cp.async segment (per warp, double-buffered)
constexpr int kPad = 8;                  // needle lists are padded to a multiple of 8 entries
constexpr int kSmallMax = 127;
constexpr int kPixBits = 14;             // pixel index bits (N <= 128)

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------- a10: pairs (general, exact)
__global__ void __launch_bounds__(256)
crss_pairs_kernel(const uint16_t *__restrict__ needles, int64_t nn, const uint16_t *__restrict__ hay,
                  int64_t nh, int N, const int64_t *__restrict__ pairs, int64_t m,
                  uint64_t *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (k >= m) return;
    int64_t i = k, j = k;
    if (pairs) { i = pairs[2 * k]; j = pairs[2 * k + 1]; }
    if (i < 0 || i >= nn || j < 0 || j >= nh) {
        if (lane == 0) out[k] = ~0ull;
        return;
    }
    const int64_t P = (int64_t)N * N;
    const uint16_t *a = needles + i * P, *b = hay + j * P;
    uint64_t acc = 0;
    if ((N % 8) == 0 && ((reinterpret_cast<uintptr_t>(needles) | reinterpret_cast<uintptr_t>(hay)) & 15) == 0) {
        // 8 pixels per lane per step (16-byte loads); the left neighbour of a run is the
        // previous lane's last pixel (P:497 shuffle), or the row's own first pixel at column 0
        for (int64_t base = 0; base < P; base += 256) {       // warp-uniform trip count
            const int64_t p0 = base + 8 * lane;
            const bool live = p0 < P;
            uint4 wa = make_uint4(0, 0, 0, 0), wb = make_uint4(0, 0, 0, 0);
            if (live) {
                wa = __ldg(reinterpret_cast<const uint4 *>(a + p0));
                wb = __ldg(reinterpret_cast<const uint4 *>(b + p0));
            }
            const unsigned pa = __shfl_up_sync(0xffffffffu, wa.w, 1), pb = __shfl_up_sync(0xffffffffu, wb.w, 1);
            if (!live) continue;
            int xa[8] = {(int)(wa.x & 0xffff), (int)(wa.x >> 16), (int)(wa.y & 0xffff), (int)(wa.y >> 16),
                         (int)(wa.z & 0xffff), (int)(wa.z >> 16), (int)(wa.w & 0xffff), (int)(wa.w >> 16)};
            int xb[8] = {(int)(wb.x & 0xffff), (int)(wb.x >> 16), (int)(wb.y & 0xffff), (int)(wb.y >> 16),
                         (int)(wb.z & 0xffff), (int)(wb.z >> 16), (int)(wb.w & 0xffff), (int)(wb.w >> 16)};
            int la, lb;
            if (p0 % N == 0) { la = xa[0]; lb = xb[0]; }
            else if (lane == 0) { la = a[p0 - 1]; lb = b[p0 - 1]; }
            else { la = (int)(pa >> 16); lb = (int)(pb >> 16); }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int64_t dn = (int64_t)xa[k] - (k ? xa[k - 1] : la);
                if (dn == 0) continue;                   // only where the needle changes
                const int64_t dh = (int64_t)xb[k] - (k ? xb[k - 1] : lb);
                acc += (uint64_t)((dn - dh) * (dn - dh));
            }
        }
    } else {
        for (int p = lane; p < P; p += 32) {
            if (p % N == 0) continue;                    // "Skip first column" (Listing 1)
            int64_t dn = (int64_t)a[p] - (int64_t)a[p - 1];
            if (dn == 0) continue;                       // only where the needle changes
            int64_t dh = (int64_t)b[p] - (int64_t)b[p - 1];
            int64_t d = dn - dh;
            acc += (uint64_t)(d * d);
        }
    }
    acc = warp_sum_u64(acc);
    if (lane == 0) out[k] = acc;
}

// ---------------------------------------------------------------- a9: needle change lists
// CSR lists: needle i's entries occupy [off[i], off[i+1]), (D_n << 14) | pixel (c >= 1) in pixel
// order, then zero entries (D_n 0, pixel 0: column 0 has D_h = 0, the term is 0) and a final
// MARKER entry (D_n 0, pixel N: column 0 of row 1, also a zero term) -- the list length is
// the smallest multiple of 8 that leaves room for the marker.  A real entry never has a
// pixel in column 0, so the marker is unambiguous.
__device__ __forceinline__ int needle_delta(const uint16_t *a, int p, int N, unsigned &mx) {
    unsigned v = a[p];
    mx = max(mx, v);
    return (p % N != 0) ? (int)v - (int)a[p - 1] : 0;
}

__global__ void __launch_bounds__(256)
needle_count_kernel(const uint16_t *__restrict__ needles, int64_t nn, int N,
                    int64_t *__restrict__ plen, int *__restrict__ n_entries,
                    unsigned char *__restrict__ small) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= nn) return;
    const int P = N * N;
    const uint16_t *a = needles + i * (int64_t)P;
    int cnt = 0;
    unsigned mx = 0;
    for (int base = 0; base < P; base += 32) {
        int dn = (base + lane < P) ? needle_delta(a, base + lane, N, mx) : 0;
        cnt += __popc(__ballot_sync(0xffffffffu, dn != 0));
    }
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
        n_entries[i] = cnt;
        plen[i] = ((cnt + 1 + kPad - 1) / kPad) * kPad;
        small[i] = mx <= (unsigned)kSmallMax;
    }
}

// exclusive scan of n int64 values in place (one CTA sweeping 1024 at a time); off[n] = total
__global__ void __launch_bounds__(1024) scan_i64_kernel(int64_t *__restrict__ v, int64_t n) {
    __shared__ int64_t part[1024];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < n; base += 1024) {
        const int64_t i = base + threadIdx.x;
        const int64_t x = i < n ? v[i] : 0;
        part[threadIdx.x] = x;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            int64_t t = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
            __syncthreads();
            part[threadIdx.x] += t;
            __syncthreads();
        }
        const int64_t incl = part[threadIdx.x] + carry;
        if (i < n) v[i] = incl - x;
        __syncthreads();
        if (threadIdx.x == 1023) carry = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) v[n] = carry;
}

__global__ void __launch_bounds__(256)
needle_fill_kernel(const uint16_t *__restrict__ needles, int64_t nn, int N,
                   const int64_t *__restrict__ off, int *__restrict__ entries) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= nn) return;
    const int P = N * N;
    const uint16_t *a = needles + i * (int64_t)P;
    int *dst = entries + off[i];
    const int len = (int)(off[i + 1] - off[i]);
    // entries in decreasing-|D_n| buckets (the sum is order-independent; large terms first make
    // the rank-mode early exit trigger sooner)
    const int lo_b[5] = {8, 4, 3, 2, 1}, hi_b[5] = {1 << 30, 7, 3, 2, 1};
    int cnt = 0;
    unsigned mx = 0;
    for (int bk = 0; bk < 5; ++bk) {
        for (int base = 0; base < P; base += 32) {
            int p = base + lane;
            int dn = (p < P) ? needle_delta(a, p, N, mx) : 0;
            const int ad = abs(dn);
            const bool take = dn != 0 && ad >= lo_b[bk] && ad <= hi_b[bk];
            unsigned m = __ballot_sync(0xffffffffu, take);
            if (take) dst[cnt + __popc(m & ((1u << lane) - 1u))] = dn * (1 << kPixBits) + p;
            cnt += __popc(m);
        }
    }
    for (int e = cnt + lane; e < len; e += 32) dst[e] = (e == len - 1) ? N : 0;
}

// ---------------------------------------------------------------- a11 + a12: tiles
struct TileArgs {
    const uint16_t *hay; int64_t nh;
    int64_t nn;
    const int *entries; const int64_t *off; const int *n_entries; const unsigned char *small;
    const uint64_t *thr; uint32_t *counts; uint64_t *dist;
    int N, plane_bytes, use_smem, early_exit;
    int64_t n_tiles, n_groups, tiles_per_group, n_items;
    unsigned long long *work;
};

__device__ __forceinline__ unsigned pack4(int a, int b, int c, int d) {
    return (unsigned)(a & 0xff) | ((unsigned)(b & 0xff) << 8) | ((unsigned)(c & 0xff) << 16) |
           ((unsigned)d << 24);
}

// One masked Eq. 7 term for this lane's haystack image: (D_n - D_h)^2.  Planes have a
// power-of-two stride S and are XOR-swizzled at 4-byte granularity by the image index, so
// the shared address of pixel p in lane j's plane is (p & (S-1)) ^ key_j with
// key_j = (tile_base + j*S) | (j << 2): one LOP3, and the 32 lanes hit 32 distinct banks.
__device__ __forceinline__ int sq_term(int entry, unsigned mask, unsigned key) {
    int dh;
    asm volatile("ld.shared.s8 %0, [%1];" : "=r"(dh) : "r"(((unsigned)entry & mask) ^ key));
    int d = (entry >> kPixBits) - dh;
    return d * d;
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Exact uint64 CRSS of needle list L (n entries) against haystack image h, from global memory.
__device__ __forceinline__ uint64_t crss_exact(const int *__restrict__ L, int n, const uint16_t *__restrict__ h) {
    uint64_t acc = 0;
    for (int e = 0; e < n; ++e) {
        int v0 = __ldg(L + e);
        int p = v0 & ((1 << kPixBits) - 1);
        int64_t dn = v0 >> kPixBits;
        int64_t dhv = (int64_t)__ldg(h + p) - (int64_t)__ldg(h + p - 1);
        int64_t df = dn - dhv;
        acc += (uint64_t)(df * df);
    }
    return acc;
}

// Close needle il for this lane's haystack image (a12): count it when CRSS < t_i (warp ballot +
// popc into the chunk's shared counters), or write the distance row.  Needles or tiles with
// a pixel above 127 take the exact 64-bit path here.  Kept out of line: it runs once per
// (needle, tile) and would otherwise crowd the registers of the entry loop.
__device__ __noinline__ void finish_needle(const TileArgs &A, int il, int64_t i0, unsigned acc, bool tsmall,
                                           bool valid, int64_t gj, const uint16_t *hj, unsigned *cnt_s,
                                           const unsigned *small_s, const uint64_t *thr_s, int lane) {
    const int64_t gi = i0 + il;
    uint64_t d = acc;
    if (!((small_s[il >> 5] >> (il & 31)) & 1u) || !tsmall)
        d = valid ? crss_exact(A.entries + A.off[gi], A.n_entries[gi], hj) : 0;
    if (A.thr) {
        unsigned bm = __ballot_sync(0xffffffffu, valid && d < thr_s[il]);
        if (lane == 0) cnt_s[il] += __popc(bm);
    }
    if (A.dist && valid) A.dist[gi * A.nh + gj] = d;
}

__global__ void __launch_bounds__(kCrssThreads, 1)
crss_tile_kernel(TileArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    // [32][S] int8 planes, S = A.plane_bytes (power of two), aligned to S in the shared window
    const unsigned S = (unsigned)A.plane_bytes;
    const unsigned raw_sh = (unsigned)__cvta_generic_to_shared(smem_raw);
    const unsigned pad = S ? ((S - (raw_sh & (S - 1))) & (S - 1)) : 0u;
    unsigned char *dh = smem_raw + pad;
    const unsigned tile_sh = raw_sh + pad;
    unsigned char *after = smem_raw + (S ? S : 16) + kTileImages * S;
    int *segbuf_all = reinterpret_cast<int *>(after);                               // [warps][2][kSeg]
    uint64_t *thr_s = reinterpret_cast<uint64_t *>(after + kWarps * 2 * kSeg * sizeof(int));  // [chunk]
    int *off_s = reinterpret_cast<int *>(thr_s + kNeedleChunk);   // [chunk+1] list offsets relative to the chunk
    __shared__ unsigned cnt_s[kNeedleChunk];
    __shared__ unsigned small_s[kNeedleChunk / 32];
    __shared__ int warp_first[kWarps + 1];
    __shared__ long long item_s;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = A.N, P = N * N;
    int *seg0 = segbuf_all + warp * 2 * kSeg;
    // 16-byte staging loads need N % 8 == 0 and a 16-byte aligned haystack base
    const bool vec_stage = (N % 8) == 0 && (reinterpret_cast<uintptr_t>(A.hay) & 15) == 0;

    for (;;) {
        __syncthreads();
        if (tid == 0) item_s = (long long)atomicAdd(A.work, 1ull);
        __syncthreads();
        const long long item = item_s;
        if (item >= A.n_items) break;
        const int64_t chunk = item / A.n_groups, group = item % A.n_groups;
        const int64_t i0 = chunk * kNeedleChunk;
        const int nc = (int)min((int64_t)kNeedleChunk, A.nn - i0);
        const int64_t t_begin = group * A.tiles_per_group;
        const int64_t t_end = min(A.n_tiles, t_begin + A.tiles_per_group);
        for (int i = tid; i <= nc; i += kCrssThreads) {
            off_s[i] = (int)(A.off[i0 + i] - A.off[i0]);
            if (i < nc) {
                cnt_s[i] = 0;
                if (A.thr) thr_s[i] = A.thr[i0 + i];
            }
        }
        for (int w = tid; w < kNeedleChunk / 32; w += kCrssThreads) {
            unsigned bits = 0;
            for (int b = 0; b < 32; ++b) {
                int i = w * 32 + b;
                if (i < nc && A.small[i0 + i]) bits |= 1u << b;
            }
            small_s[w] = bits;
        }
        // split the chunk's entry stream into kWarps runs of whole needles with ~equal entries
        if (tid <= kWarps) {
            const int64_t e0 = A.off[i0], e1 = A.off[i0 + nc];
            const int64_t target = e0 + (e1 - e0) * tid / kWarps;
            int lo = 0, hi = nc;                         // first needle with off >= target
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if (A.off[i0 + mid] < target) lo = mid + 1; else hi = mid;
            }
            warp_first[tid] = tid == kWarps ? nc : (tid == 0 ? 0 : lo);
        }
        __syncthreads();
        const int wa = warp_first[warp], wb = max(wa, warp_first[warp + 1]);
        const int64_t s_begin = A.off[i0 + wa], s_end = A.off[i0 + wb];
        const int n_seg = (int)((s_end - s_begin + kSeg - 1) / kSeg);

        for (int64_t tile = t_begin; tile < t_end; ++tile) {
            const int64_t j0 = tile * kTileImages;
            const int nj = (int)min((int64_t)kTileImages, A.nh - j0);
            __syncthreads();                              // previous tile fully consumed
            // first segment of this warp's needle stream: overlaps with the tile staging
            if (n_seg > 0 && lane * 4 < kSeg && s_begin + lane * 4 < s_end)
                cp_async16(seg0 + lane * 4, A.entries + s_begin + lane * 4);
            cp_async_commit();
            // stage D_h(r,c) = h[r][c] - h[r][c-1] as int8 planes (0 in column 0); the left
            // neighbour of a thread's 8-pixel run comes from the previous lane
            int small_local = 1;
            if (A.use_smem) {
                if (vec_stage) {
                    const int runs = P / 8;               // per image
                    for (int q0 = 0; q0 < kTileImages * runs; q0 += kCrssThreads) {
                        const int q = q0 + tid;
                        const int j = q / runs, p = (q - j * runs) * 8;
                        uint4 w = make_uint4(0, 0, 0, 0);
                        const bool live = (q < kTileImages * runs) && j < nj;
                        if (live) w = __ldg(reinterpret_cast<const uint4 *>(A.hay + (j0 + j) * (int64_t)P + p));
                        unsigned prev_hi = __shfl_up_sync(0xffffffffu, w.w, 1);
                        int left;
                        if (p % N == 0) left = (int)(w.x & 0xffff);          // column 0: D_h = 0
                        else if (lane == 0) left = live ? (int)__ldg(A.hay + (j0 + j) * (int64_t)P + p - 1) : 0;
                        else left = (int)(prev_hi >> 16);
                        int x[8] = {(int)(w.x & 0xffff), (int)(w.x >> 16), (int)(w.y & 0xffff), (int)(w.y >> 16),
                                    (int)(w.z & 0xffff), (int)(w.z >> 16), (int)(w.w & 0xffff), (int)(w.w >> 16)};
                        int mx = max(max(max(x[0], x[1]), max(x[2], x[3])), max(max(x[4], x[5]), max(x[6], x[7])));
                        small_local &= (mx <= kSmallMax);
                        if (q < kTileImages * runs) {
                            unsigned char *pl = dh + j * S;
                            const unsigned key = (unsigned)j << 2;
                            *reinterpret_cast<unsigned *>(pl + ((unsigned)p ^ key)) =
                                pack4(x[0] - left, x[1] - x[0], x[2] - x[1], x[3] - x[2]);
                            *reinterpret_cast<unsigned *>(pl + ((unsigned)(p + 4) ^ key)) =
                                pack4(x[4] - x[3], x[5] - x[4], x[6] - x[5], x[7] - x[6]);
                        }
                    }
                } else {
                    for (int q = tid; q < kTileImages * P; q += kCrssThreads) {
                        int j = q / P, p = q - j * P;
                        int v = 0;
                        if (j < nj) {
                            const uint16_t *h = A.hay + (j0 + j) * (int64_t)P;
                            int x = __ldg(h + p);
                            int xl = (p % N) ? (int)__ldg(h + p - 1) : x;
                            small_local &= (x <= kSmallMax);
                            v = x - xl;
                        }
                        dh[j * S + ((unsigned)p ^ ((unsigned)j << 2))] = (unsigned char)(signed char)v;
                    }
                }
            } else {
                small_local = 0;
            }
            const int tile_small = __syncthreads_and(small_local);

            const unsigned mask = S - 1u;
            const unsigned key = (tile_sh + (unsigned)lane * S) | ((unsigned)lane << 2);
            const bool valid = lane < nj;
            const int64_t gj = j0 + lane;
            const uint16_t *hj = A.hay + (valid ? gj : j0) * (int64_t)P;

            const bool tsmall = tile_small != 0;
            if (!tile_small) {
                cp_async_wait<0>();
                for (int il = wa; il < wb; ++il) finish_needle(A, il, i0, 0, tsmall, valid, gj, hj, cnt_s, small_s, thr_s, lane);
                continue;
            }
            // fast path: the warp's stream in double-buffered segments, consumed in runs that
            // end at a needle boundary or a segment boundary (both multiples of 8 entries)
            int il = wa;
            int rem = wa < wb ? off_s[wa + 1] - off_s[wa] : 0;
            unsigned acc = 0;
            const bool early = A.early_exit != 0;
            bool dead = false;                                // rank mode: every lane already >= t_i
            uint64_t t_cur = (early && wa < wb) ? thr_s[wa] : 0;
            for (int k = 0; k < n_seg; ++k) {
                if (k + 1 < n_seg) {
                    const int64_t nb = s_begin + (int64_t)(k + 1) * kSeg;
                    int *dst = seg0 + ((k + 1) & 1) * kSeg;
                    if (lane * 4 < kSeg && nb + lane * 4 < s_end) cp_async16(dst + lane * 4, A.entries + nb + lane * 4);
                    cp_async_commit();
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
                __syncwarp();
                const int *buf = seg0 + (k & 1) * kSeg;
                const int len = (int)min((int64_t)kSeg, s_end - s_begin - (int64_t)k * kSeg);
                int e = 0;
                while (e < len) {
                    const int run = min(rem, len - e);
                    const int *b = buf + e;
                    if (!early) {
#pragma unroll 2
                        for (int q = 0; q < run; q += kPad) {
                            const int4 u = *reinterpret_cast<const int4 *>(b + q);
                            const int4 v = *reinterpret_cast<const int4 *>(b + q + 4);
                            acc += (unsigned)(sq_term(u.x, mask, key) + sq_term(u.y, mask, key) + sq_term(u.z, mask, key) + sq_term(u.w, mask, key));
                            acc += (unsigned)(sq_term(v.x, mask, key) + sq_term(v.y, mask, key) + sq_term(v.z, mask, key) + sq_term(v.w, mask, key));
                        }
                    } else if (!dead) {
                        // partial sums only grow, so once every lane is >= t_i the
                        // needle's remaining terms cannot change any count (G12)
                        for (int q = 0; q < run; q += kPad) {
                            const int4 u = *reinterpret_cast<const int4 *>(b + q);
                            const int4 v = *reinterpret_cast<const int4 *>(b + q + 4);
                            acc += (unsigned)(sq_term(u.x, mask, key) + sq_term(u.y, mask, key) + sq_term(u.z, mask, key) + sq_term(u.w, mask, key));
                            acc += (unsigned)(sq_term(v.x, mask, key) + sq_term(v.y, mask, key) + sq_term(v.z, mask, key) + sq_term(v.w, mask, key));
                            if (__all_sync(0xffffffffu, !valid || (uint64_t)acc >= t_cur)) { dead = true; break; }
                        }
                    }
                    e += run;
                    rem -= run;
                    if (rem == 0) {
                        finish_needle(A, il, i0, acc, tsmall, valid, gj, hj, cnt_s, small_s, thr_s, lane);
                        acc = 0;
                        dead = false;
                        ++il;
                        rem = il < wb ? off_s[il + 1] - off_s[il] : 0;
                        if (early && il < wb) t_cur = thr_s[il];
                    }
                }
                __syncwarp();
            }
        }
        __syncthreads();
        if (A.thr)
            for (int i = tid; i < nc; i += kCrssThreads)
                if (cnt_s[i]) atomicAdd(A.counts + i0 + i, cnt_s[i]);
    }
}

}  // namespace

cudaError_t launch_crss_pairs(const uint16_t *d_needles, int64_t nn, const uint16_t *d_haystack,
                              int64_t nh, int N, const int64_t *d_pairs, int64_t m,
                              uint64_t *d_out, cudaStream_t s) {
    if (m == 0) return cudaSuccess;
    const int warps = 8;
    int64_t blocks = (m + warps - 1) / warps;
    crss_pairs_kernel<<<(unsigned)blocks, 32 * warps, 0, s>>>(d_needles, nn, d_haystack, nh, N,
                                                              d_pairs, m, d_out);
    note_launches(1);
    return cudaGetLastError();
}

cudaError_t launch_crss_search_tiles(const uint16_t *d_needles, int64_t nn,
                                     const uint16_t *d_haystack, int64_t nh, int N,
                                     const uint64_t *d_thresholds, uint32_t *d_counts,
                                     uint64_t *d_dist, cudaStream_t s, bool early_exit) {
    cudaError_t e;
    if (d_counts && nn > 0) {
        e = cudaMemsetAsync(d_counts, 0, sizeof(uint32_t) * nn, s);
        if (e != cudaSuccess) return e;
    }
    if (nn == 0 || nh == 0) return cudaSuccess;
    const int P = N * N;
    // a9: CSR needle change lists
    int64_t *off = nullptr;
    int *n_entries = nullptr, *entries = nullptr;
    unsigned char *small = nullptr;
    unsigned long long *work = nullptr;
    if ((e = cudaMallocAsync((void **)&off, sizeof(int64_t) * (nn + 1), s)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync((void **)&n_entries, sizeof(int) * nn, s)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync((void **)&small, nn, s)) != cudaSuccess) return e;
    if ((e = cudaMallocAsync((void **)&work, sizeof(unsigned long long), s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(work, 0, sizeof(unsigned long long), s)) != cudaSuccess) return e;
    const int warps = 8;
    const unsigned nb = (unsigned)((nn + warps - 1) / warps);
    needle_count_kernel<<<nb, 32 * warps, 0, s>>>(d_needles, nn, N, off, n_entries, small);
    scan_i64_kernel<<<1, 1024, 0, s>>>(off, nn);
    note_launches(2);
    // the list sizes are only known on the device: allocate the worst case
    // (N(N-1) deltas + marker, rounded to 8, per needle) -- stream-ordered, pooled
    const int64_t cap = ((int64_t)N * (N - 1) + 1 + kPad - 1) / kPad * kPad;
    if ((e = cudaMallocAsync((void **)&entries, sizeof(int) * cap * nn, s)) != cudaSuccess) return e;
    needle_fill_kernel<<<nb, 32 * warps, 0, s>>>(d_needles, nn, N, off, entries);
    note_launches(1);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;

    TileArgs A;
    A.hay = d_haystack; A.nh = nh; A.nn = nn;
    A.entries = entries; A.off = off; A.n_entries = n_entries; A.small = small;
    A.thr = d_thresholds; A.counts = d_counts; A.dist = d_dist;
    A.N = N;
    A.early_exit = (early_exit && d_thresholds && !d_dist) ? 1 : 0;
    int stride = 128;                                    // power of two >= P (XOR swizzle needs >= 128)
    while (stride < P) stride <<= 1;
    A.plane_bytes = stride;
    size_t smem = (size_t)(kTileImages + 1) * stride;    // + alignment slack
    A.use_smem = (kTileImages * (size_t)stride <= 128 * 1024) && P < (1 << kPixBits);
    if (!A.use_smem) { smem = 16; A.plane_bytes = 0; }
    smem += (size_t)kWarps * 2 * kSeg * sizeof(int) + (size_t)kNeedleChunk * sizeof(uint64_t) +
            (size_t)(kNeedleChunk + 1) * sizeof(int);
    A.n_tiles = (nh + kTileImages - 1) / kTileImages;
    int64_t n_chunks = (nn + kNeedleChunk - 1) / kNeedleChunk;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t want = 4LL * sms;
    int64_t groups = (want + n_chunks - 1) / n_chunks;
    if (groups < 1) groups = 1;
    if (groups > A.n_tiles) groups = A.n_tiles;
    A.tiles_per_group = (A.n_tiles + groups - 1) / groups;
    A.n_groups = (A.n_tiles + A.tiles_per_group - 1) / A.tiles_per_group;
    A.n_items = n_chunks * A.n_groups;
    A.work = work;
    if ((e = ensure_smem((const void *)crss_tile_kernel, smem)) != cudaSuccess) return e;
    int64_t grid = A.n_items < sms ? A.n_items : sms;
    crss_tile_kernel<<<(unsigned)grid, kCrssThreads, smem, s>>>(A);
    note_launches(1);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    cudaFreeAsync(entries, s);
    cudaFreeAsync(off, s);
    cudaFreeAsync(n_entries, s);
    cudaFreeAsync(small, s);
    cudaFreeAsync(work, s);
    return cudaSuccess;
}

}  // namespace rici

/*
 * rici.h -- C ABI of the B200-native RICI hot path (arXiv 2007.02306).
 *
 * Two steps of the paper's method run behind this boundary, as hand-written
 * sm_100a CUDA kernels:
 *   (a) RICI construction   "iterate over each triangle in the scene",
 *       three steps per triangle: project (Eqs. 1-5),
 *       per-layer circle/triangle intersection ranges, bin increments.
 *   (b) CRSS search         the clutter-resistant distance (Eq. 6, Eq. 7
 *       P:346-348, Listing 1) of every needle against every haystack
 *       image, and the rank of the true correspondence (best tie P:459).
 * "P:n" = line n of the paper text; G1..G16 = readings listed in DESIGN.md.
 *
 * Conventions for every entry point
 * ---------------------------------
 * Pointers.  Every bulk pointer may be CUDA DEVICE memory or HOST memory
 *   (pinned or pageable); the library inspects it with cudaPointerGetAttributes.
 *   Host inputs are copied to device workspace on `stream`; host outputs are
 *   copied back on `stream` and the call then synchronises `stream` before it
 *   returns.  With device pointers nothing is synchronised (except
 *   rici_create_mesh, see there).
 * Ownership.  The caller owns every buffer it passes; the library never frees
 *   or retains them past the call.  Inputs are never modified.  A rici_mesh
 *   owns its device triangle buffer until rici_destroy_mesh.
 * Stream.  All work is enqueued on `stream` (a cudaStream_t; NULL = legacy
 *   default stream) on the current device.  Outputs on device are valid once
 *   the stream reaches the point of the call.
 * Errors.  Each call returns a rici_status.  Argument errors are detected
 *   synchronously before anything is enqueued (RICI_ERR_INVALID_ARGUMENT).
 *   CUDA errors return RICI_ERR_CUDA.  A device other than sm_100 returns
 *   RICI_ERR_UNSUPPORTED.  rici_last_error() gives a message for the last
 *   failing call on the calling thread.  No exception or abort crosses the ABI.
 * Images.  A RICI image is n_bins x n_bins uint16, row-major
 *   [row = beta layer, ascending][column = radius alpha, ascending] (P:117-121,
 *   G4), counts saturated at 65535 (G9).  2 <= n_bins <= 128 is accepted;
 *   n_bins = 64 is the paper's setting and the tuned path.
 */
#ifndef RICI_H_
#define RICI_H_

#include <stdint.h>

#if defined(__GNUC__)
#define RICI_API __attribute__((visibility("default")))
#else
#define RICI_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *rici_stream_t;   /* identical to cudaStream_t */
typedef struct rici_mesh_s *rici_mesh;       /* opaque device triangle buffer */

typedef enum {
    RICI_OK = 0,
    RICI_ERR_INVALID_ARGUMENT = 1,
    RICI_ERR_CUDA = 2,
    RICI_ERR_OUT_OF_MEMORY = 3,
    RICI_ERR_UNSUPPORTED = 4
} rici_status;

/* ---- (a1) mesh staging ----------------------------------------------------
 * Builds the device triangle buffer the construction kernel streams: every
 * triangle "in the scene" de-indexed into its three vertex positions
 * and grouped into spatially compact chunks (an internal reordering that
 * cannot change any image: counts are sums over triangles).
 *   vertices   [n_vertices][3] float32 x,y,z
 *   indices    [n_triangles][3] int32, each in [0, n_vertices)
 *   out_mesh   receives the handle (unchanged on error)
 * n_triangles = 0 is a valid empty scene (every image is zero); at most 268,435,456
 * triangles (RICI_ERR_INVALID_ARGUMENT beyond).
 * Index validation reads the indices, so this call synchronises `stream` once (after the
 * validating first pass); an out-of-range index returns RICI_ERR_INVALID_ARGUMENT.  The
 * spatial sort and chunk staging that follow run asynchronously on `stream`: a use of the mesh
 * on another stream first waits for them (an event recorded by this call), and
 * rici_destroy_mesh waits for them too.                                       */
RICI_API rici_status rici_create_mesh(const float *vertices, int64_t n_vertices,
                             const int32_t *indices, int64_t n_triangles,
                             rici_stream_t stream, rici_mesh *out_mesh);

/* Frees the mesh: stream-ordered release on the legacy default stream, made to wait for the
 * last rici_generate / rici_clutter_fraction that read the mesh on every stream it was used on
 * (blocking or non-blocking); does not block the host.  The handle is invalid afterwards.
 * NULL is a no-op. */
RICI_API rici_status rici_destroy_mesh(rici_mesh mesh);

/* Number of triangles in the mesh, or -1 for NULL. */
RICI_API int64_t rici_mesh_num_triangles(rici_mesh mesh);

/* ---- (a2-a8) RICI construction ---------------------------------------------
 * One RICI per oriented point (spin vertex S_v + spin normal S_n).
 *   origins        [n][6] float32 (px,py,pz,nx,ny,nz); the normal need not be
 *                  unit length (it is normalised, G3); a zero or non-finite
 *                  normal yields an all-zero image (not an error).
 *   n              >= 0 images
 *   support_radius R > 0, finite: image width R (alpha in [0,R]) and height R
 *                  (beta in [-R/2, R/2]) (G4)
 *   n_bins         N in [2,128]
 *   out            [n][N][N] uint16, fully overwritten
 * Arithmetic is FP32 (paper: float kernels, G13); pixels whose circle lies
 * within ~1e-5*R of a layer/bin/sign decision may differ from an exact
 * evaluation (the north-star attribution rule).                             */
RICI_API rici_status rici_generate(rici_mesh mesh, const float *origins, int64_t n,
                          float support_radius, int32_t n_bins,
                          uint16_t *out, rici_stream_t stream);

/* ---- (a9-a12) CRSS search ---------------------------------------------------
 * Rank of each needle's true correspondence with the implicit correspondence
 * needle i <-> haystack i (G11): rank_i = #{ j : CRSS(n_i,h_j) < CRSS(n_i,h_i) }
 * (strict, so ties take the best rank; 0 <= rank <= n_haystack-1).
 *   needles    [n_needles][N][N] uint16
 *   haystack   [n_haystack][N][N] uint16, n_haystack >= n_needles
 *   out_ranks  [n_needles] uint32
 * Exact integer arithmetic (bit-exact for every input).
 * Kernels: for n_bins = 64 the counts run on the tensor cores (tcgen05 int8 GEMM of the
 * expanded Eq. 7, exact under a per-image guard |D_n| <= 63, |D_h| <= 15) and the pairs with an
 * image outside the guard are counted exactly by fallback kernels sized on the device (see
 * rici_crss_guard_stats).  Other n_bins, or RICI_CRSS_PATH=simt in the environment, use the SIMT
 * kernel only.  No path synchronises the host (device buffers; the calls can be captured in a
 * CUDA graph).  Temporary workspace is stream-ordered (cudaMallocAsync) and, at n_bins = 64,
 * about 2 x 8 KB per needle row plus 8 KB per haystack row.  rici_crss_count_below follows the
 * same rules.                                                                             */
RICI_API rici_status rici_crss_search(const uint16_t *needles, int64_t n_needles,
                             const uint16_t *haystack, int64_t n_haystack,
                             int32_t n_bins, uint32_t *out_ranks, rici_stream_t stream);

/* rici_crss_search with options.  flags:
 *   RICI_CRSS_SIMT        use the SIMT kernel even for n_bins = 64 (no synchronisation)
 *   RICI_CRSS_EARLY_EXIT  rank mode ("cease execution when a predetermined distance
 *                         threshold is exceeded").  Every CRSS term is a square, so the sum
 *                         over any subset of pixels is a lower bound and stopping once it is
 *                         >= t_i leaves the ranks identical (G12).
 *                         Tensor path (n_bins = 64): two prune-check passes over the K prefixes
 *                         of image rows 24-39 and 16-47 retire every 256 x 256 tile whose
 *                         guard-valid pairs are all >= t_i; the survivors run the full K.
 *                         With RICI_CRSS_SIMT: a needle's accumulation over a group of 32
 *                         haystack images stops once every partial sum is >= t_i (needle
 *                         entries visited in decreasing |D_n|).                             */
#define RICI_CRSS_SIMT 1u
#define RICI_CRSS_EARLY_EXIT 2u
RICI_API rici_status rici_crss_search_ex(const uint16_t *needles, int64_t n_needles,
                                         const uint16_t *haystack, int64_t n_haystack,
                                         int32_t n_bins, uint32_t flags, uint32_t *out_ranks,
                                         rici_stream_t stream);

/* Sharding primitives (used by the multi-GPU layer).
 * rici_crss_pairs: out[k] = CRSS(needles[pairs[k][0]], haystack[pairs[k][1]]) -- Eq. 7
 *   (Listing 1) for an explicit pair list: the threshold pass a10, t_i =
 *   CRSS(n_i, h_{k_i}) ("this threshold can be trivially precomputed"; G11 for k_i), run
 *   by the rank that owns h_{k_i}.
 *   pairs [m][2] int64 (needle index, haystack index).  With HOST pairs every
 *   index is validated (RICI_ERR_INVALID_ARGUMENT); with DEVICE pairs an
 *   out-of-range pair yields out[k] = UINT64_MAX.                           */
RICI_API rici_status rici_crss_pairs(const uint16_t *needles, int64_t n_needles,
                            const uint16_t *haystack, int64_t n_haystack, int32_t n_bins,
                            const int64_t *pairs, int64_t m, uint64_t *out,
                            rici_stream_t stream);

/* out_counts[i] = #{ j in [0,n_haystack) : CRSS(needles[i], haystack[j]) < thresholds[i] }
 * (overwritten, not accumulated).  thresholds [n_needles] uint64.  With t_i = CRSS(n_i, h_i)
 * this is the rank of P:388 ("lower ranks are better") with the best-tie rule of P:459 (strict
 * <, G10) restricted to one haystack shard; the per-shard counts of all ranks sum to the rank. */
RICI_API rici_status rici_crss_count_below(const uint16_t *needles, int64_t n_needles,
                                  const uint16_t *haystack, int64_t n_haystack, int32_t n_bins,
                                  const uint64_t *thresholds, uint32_t *out_counts,
                                  rici_stream_t stream);

/* Full distance matrix out[i][j] = CRSS(needles[i], haystack[j]), uint64: Eq. 7,
 * exact, asymmetric in its arguments (only the needle's changes are masked). SIMT kernel. */
RICI_API rici_status rici_crss_distances(const uint16_t *needles, int64_t n_needles,
                                const uint16_t *haystack, int64_t n_haystack, int32_t n_bins,
                                uint64_t *out, rici_stream_t stream);

/* ---- (f4) clutter fraction, Eq. 8 ---------------------------------
 * clutter = (A_all - A_object) / A_all per oriented point, A over the support volume (the
 * RICI cylinder r <= R, |beta| <= R/2; G17).  Areas by a fixed quadrature: every triangle
 * is cut into Q x Q congruent sub-triangles and a sub-triangle counts (area A/Q^2) when its
 * centroid is inside.  0 when no surface is inside.
 *   object_tag      [n_triangles] uint8 in the caller's triangle order (the order given to
 *                   rici_create_mesh): non-zero = part of the object of interest
 *   origins         [n][6] float32 as for rici_generate
 *   quadrature_q    Q in [1, 16]
 *   out_fraction    [n] float32
 *   out_area_all    [n] float32 A_all, or NULL                                       */
RICI_API rici_status rici_clutter_fraction(rici_mesh mesh, const uint8_t *object_tag,
                                           const float *origins, int64_t n, float support_radius,
                                           int32_t quadrature_q, float *out_fraction,
                                           float *out_area_all, rici_stream_t stream);

/* ---- diagnostics ------------------------------------------------------------ */
/* Message of the last failing call on this thread ("" if none).  Valid until
 * the next rici_* call on this thread. */
RICI_API const char *rici_last_error(void);

/* Total number of kernels this library has launched in this process. */
RICI_API uint64_t rici_launch_count(void);

/* Per-kernel device timing (for the roofline: a kernel's own launch durations, measured live
 * with CUDA events recorded on the stream each launch is issued to).  Off by default; while
 * on, every launch of the timed kernels records an event pair (a few microseconds of host
 * work, no device synchronisation).
 *   kernel  RICI_KERNEL_GENERATE   the construction kernel of rici_generate
 *           RICI_KERNEL_CRSS_MMA   the tcgen05 GEMM launch(es) of one count / search call
 *                                  (rank mode: all its passes together)
 * rici_kernel_time_ms waits for the recorded events, writes the mean device time in ms per
 * API call (the durations of all of that call's timed launches summed; 0 if none) and the
 * number of recorded launches, and clears the record.  Errors:
 * RICI_ERR_INVALID_ARGUMENT for an unknown kernel id or NULL output.                    */
#define RICI_KERNEL_GENERATE 0
#define RICI_KERNEL_CRSS_MMA 1
RICI_API rici_status rici_set_kernel_timing(int32_t enable);
RICI_API rici_status rici_kernel_time_ms(int32_t kernel, float *out_mean_ms, int64_t *out_launches);

/* Guard coverage of the tensor-core CRSS path (n_bins = 64) on the current device, accumulated
 * over every count / search call since the last reset:
 *   out[0] needles                       out[1] needles outside the int8 guard (|D_n| > 63)
 *   out[2] haystack images               out[3] haystack images outside it (|D_h| > 15)
 *   out[4] guard-valid needles that are not 2:4-sparse (the dense tensor pass)
 * Pairs with an image outside the guard are counted exactly by the fallback kernels; these
 * counters say how much work took that path.  Synchronises the device.  reset != 0 zeroes the
 * counters after reading.  Errors: RICI_ERR_INVALID_ARGUMENT for a NULL out.                */
RICI_API rici_status rici_crss_guard_stats(int64_t out[5], int32_t reset);

/* "rici-b200 <version> sm_100a" */
RICI_API const char *rici_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RICI_H_ */

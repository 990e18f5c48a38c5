/*
 * rici_oracle.c -- CPU oracle for the RICI hot path (arXiv 2007.02306).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2007_02306_b200/) never imports, links or calls it,
 * and shares no code, header, table or constant with it.
 *
 * Plain, slow, obviously-correct double-precision loops that follow the paper
 * step by step.  Citations are "P:n" = line n of the paper text,
 * with the section / equation / listing the line falls in.  Readings where the
 * paper is silent or garbled are tagged G1..G16 and listed in DESIGN.md.
 *
 * Pinning status (see tests/test_oracle_*.py and DESIGN.md "Oracle pins"):
 *   spin frame + projection (Eqs. 1-5)   pinned: closed-form frame, SPEC examples,
 *                                        isometry / beta = dot invariants
 *   segment ranges (P:270-276 steps 1-6) pinned: hand-worked triangle (H2), quadratic
 *   rici_generate            pinned: cube / tetra closed forms (H3,H4),
 *                                        vertical plane (H5), watertight evenness (H8),
 *                                        independent circle-plane definition O-def (H7)
 *   rici_definition (O-def)   pinned: same closed forms as above
 *   crss (Eq. 7, Listing 1)              pinned: hand example (=5), algebraic identities
 *   ranks                 pinned: tie example, sort-based brute force
 *   clutter fraction (Eq. 8)  pinned: closed-form areas of planes through the
 *                                        support cylinder (quadrature convergence), exact
 *                                        0 / 0.5 cases, fully-inside triangles
 *   The paper prints no descriptor value, distance or rank, so no pin is a
 *   number printed in the paper ("parity unpinned" against published values).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* Spin frame: Eq. 1, with the G1 correction.                    */
/* ------------------------------------------------------------------------ */
typedef struct {
    double nax, nay;   /* N_a : first rotation, about z            (Eq. 3) */
    double nbx, nbz;   /* N_b : second rotation, about y           (Eq. 4) */
    double sv[3];      /* S_v : spin vertex                        (Eq. 2) */
    int valid;         /* 0 for a zero-length normal (G3)                  */
} frame_t;

/* Eq. 1 as printed normalises (S_nx, S_nz) for N_b; that fails for every
 * normal with S_ny != 0 (G1).  The second rotation acts on the normal AFTER
 * the first rotation, whose x component is N_ax*S_nx + N_ay*S_ny
 * (= sqrt(S_nx^2+S_ny^2)), so N_b = Normalize[that, S_nz].
 * "When both coefficients of either N_a or N_b are zero, ... an identity
 * rotation is used instead" -> N_a = (1,0) when S_nx = S_ny = 0 (G2). */
static frame_t spin_frame(const double origin[6]) {
    frame_t f;
    f.sv[0] = origin[0]; f.sv[1] = origin[1]; f.sv[2] = origin[2];
    double nx = origin[3], ny = origin[4], nz = origin[5];
    double len = sqrt(nx * nx + ny * ny + nz * nz);
    f.valid = len > 0.0;
    if (!f.valid) { f.nax = 1; f.nay = 0; f.nbx = 0; f.nbz = 1; return f; }
    nx /= len; ny /= len; nz /= len;                    /* G3: normalise S_n */
    double la = sqrt(nx * nx + ny * ny);
    if (la == 0.0) { f.nax = 1.0; f.nay = 0.0; }        /* identity */
    else { f.nax = nx / la; f.nay = ny / la; }
    double sx = f.nax * nx + f.nay * ny;                /* normal x after Eq. 3 */
    double lb = sqrt(sx * sx + nz * nz);
    f.nbx = sx / lb; f.nbz = nz / lb;
    return f;
}

/* Eqs. 2-4: translate, rotate about z, rotate about y.
 * Output T = (T_x, T_y, T_z); Eq. 5: alpha = |(T_x,T_y)|, beta = T_z. */
static void project(const frame_t *f, const double p[3], double t[3]) {
    double px = p[0] - f->sv[0];                        /* Eq. 2 */
    double py = p[1] - f->sv[1];
    double pz = p[2] - f->sv[2];
    double qx = f->nax * px + f->nay * py;              /* Eq. 3 */
    double qy = -f->nay * px + f->nax * py;
    t[0] = f->nbz * qx - f->nbx * pz;                   /* Eq. 4 */
    t[1] = qy;
    t[2] = f->nbx * qx + f->nbz * pz;
}

EXPORT int oracle_spin_frame(const double origin[6], double out[4]) {
    frame_t f = spin_frame(origin);
    out[0] = f.nax; out[1] = f.nay; out[2] = f.nbx; out[3] = f.nbz;
    return f.valid;
}

EXPORT void oracle_project(const double origin[6], const double p[3], double out[2]) {
    frame_t f = spin_frame(origin);
    double t[3];
    project(&f, p, t);
    out[0] = sqrt(t[0] * t[0] + t[1] * t[1]);           /* Eq. 5 alpha */
    out[1] = t[2];                                      /* Eq. 5 beta  */
}

/* ------------------------------------------------------------------------ */
/* Circle-triangle intersection for one layer: P:246-276 (six steps).        */
/* ------------------------------------------------------------------------ */
typedef struct {
    double e0[2], e1[2];   /* E0 on the long edge (a,c); E1 on (a,b) or (b,c)   */
    double x0, x1, y;      /* E0, E1 after the alignment rotation (step 2)      */
    double rmin, rmax;     /* single-intersection radii [rmin, rmax) (step 4)   */
    double rc;             /* |C| when a double intersection exists, else -1    */
} seg_t;

/* a, b, c: projected vertices sorted by z (a.z <= b.z <= c.z).
 * Returns 0 when the plane z = beta misses the triangle under the half-open
 * layer rule z_a <= beta < z_c (G5), or the segment has zero length. */
static int segment_ranges(const double a[3], const double b[3], const double c[3],
                          double beta, seg_t *s) {
    if (!(a[2] <= beta && beta < c[2])) return 0;       /* beta-extent */
    /* Step 1: E0 on edge (a,c), E1 on the edge the plane crosses
     * below (a,b) or above (b,c) the middle vertex.  The half-open rule makes
     * every denominator below strictly positive (G5/G6). */
    double t = (beta - a[2]) / (c[2] - a[2]);
    s->e0[0] = a[0] + t * (c[0] - a[0]);
    s->e0[1] = a[1] + t * (c[1] - a[1]);
    if (beta < b[2]) {
        double u = (beta - a[2]) / (b[2] - a[2]);
        s->e1[0] = a[0] + u * (b[0] - a[0]);
        s->e1[1] = a[1] + u * (b[1] - a[1]);
    } else {
        double u = (beta - b[2]) / (c[2] - b[2]);
        s->e1[0] = b[0] + u * (c[0] - b[0]);
        s->e1[1] = b[1] + u * (c[1] - b[1]);
    }
    /* Step 2: rotate about z so E0E1 is parallel to x; the
     * normalised direction is used directly as (cos, sin). */
    double dx = s->e1[0] - s->e0[0], dy = s->e1[1] - s->e0[1];
    double len = sqrt(dx * dx + dy * dy);
    if (len == 0.0) return 0;                           /* single point: G5 */
    double cs = dx / len, sn = dy / len;
    s->x0 = cs * s->e0[0] + sn * s->e0[1];
    s->y  = -sn * s->e0[0] + cs * s->e0[1];
    s->x1 = cs * s->e1[0] + sn * s->e1[1];
    /* Step 3: distances of E0 and E1 from the z axis. */
    double r0 = sqrt(s->e0[0] * s->e0[0] + s->e0[1] * s->e0[1]);
    double r1 = sqrt(s->e1[0] * s->e1[0] + s->e1[1] * s->e1[1]);
    /* Step 4: single range [min, max) (half-open, G5). */
    s->rmin = r0 < r1 ? r0 : r1;
    s->rmax = r0 < r1 ? r1 : r0;
    /* Steps 5-6: double intersection iff the x signs differ
     * (x = 0 counts as non-negative, G5); range [|C|, min), |C| = |y|. */
    s->rc = ((s->x0 < 0.0) != (s->x1 < 0.0)) ? fabs(s->y) : -1.0;
    return 1;
}

static void sort3_by_z(const double *p[3]) {
    /* stable sort of three vertex pointers by z */
    if (p[1][2] < p[0][2]) { const double *t = p[0]; p[0] = p[1]; p[1] = t; }
    if (p[2][2] < p[1][2]) { const double *t = p[1]; p[1] = p[2]; p[2] = t; }
    if (p[1][2] < p[0][2]) { const double *t = p[0]; p[0] = p[1]; p[1] = t; }
}

/* Public helper for the hand-worked segment example.
 * out = {E0x, E0y, E1x, E1y, rmin, rmax, |C| or -1}; returns 1 if a segment exists. */
EXPORT int oracle_segment(const double t0[3], const double t1[3], const double t2[3],
                          double beta, double out[7]) {
    const double *p[3] = {t0, t1, t2};
    sort3_by_z(p);
    seg_t s;
    if (!segment_ranges(p[0], p[1], p[2], beta, &s)) return 0;
    out[0] = s.e0[0]; out[1] = s.e0[1]; out[2] = s.e1[0]; out[3] = s.e1[1];
    out[4] = s.rmin; out[5] = s.rmax; out[6] = s.rc;
    return 1;
}

/* ------------------------------------------------------------------------ */
/* RICI generation: P:132-138 (three steps per triangle).                    */
/* ------------------------------------------------------------------------ */
/* Bin geometry (G4): Delta = R/N, row centres beta_r = (r+1/2)Delta - R/2
 * ("Spin Vertex at its vertical halfway point"; height R), column
 * radii rho_c = (c+1/2)Delta ("fixed number of radii"). */
static double row_beta(int r, double R, int N) { return (r + 0.5) * (R / N) - 0.5 * R; }
static double col_rho(int c, double R, int N) { return (c + 0.5) * (R / N); }

/* One image, evaluated with every circle displaced by (dbeta, drho).  The
 * undisplaced call (0,0) is the oracle; displaced calls feed the fragility
 * rule.  img receives exact counts (uint32, no saturation). */
static void image_counts(const frame_t *f, const float *vertices, const int32_t *indices,
                         int64_t nt, double R, int N, double dbeta, double drho,
                         uint32_t *img, int64_t *stats) {
    memset(img, 0, sizeof(uint32_t) * (size_t)N * N);
    if (!f->valid) return;                               /* G3: zero normal */
    const double delta = R / N;
    for (int64_t k = 0; k < nt; ++k) {
        /* Step 1: project the triangle vertices (Eqs. 2-4). */
        double v[3][3], t[3][3];
        for (int j = 0; j < 3; ++j) {
            const float *src = vertices + 3 * (int64_t)indices[3 * k + j];
            v[j][0] = src[0]; v[j][1] = src[1]; v[j][2] = src[2];
            project(f, v[j], t[j]);
        }
        const double *p[3] = {t[0], t[1], t[2]};
        sort3_by_z(p);
        if (stats) {
            /* counts "pairs in slab": triangles whose beta-extent meets the image height */
            if (p[2][2] > -0.5 * R + dbeta && p[0][2] < 0.5 * R + dbeta) stats[0]++;
        }
        /* Step 2: every layer beta in the triangle's beta-extent.
         * The start index is only a conservative starting point; membership
         * is decided by the exact test inside segment_ranges. */
        int r0 = (int)floor((p[0][2] - dbeta + 0.5 * R) / delta - 0.5) - 1;
        if (r0 < 0) r0 = 0;
        for (int r = r0; r < N; ++r) {
            double beta = row_beta(r, R, N) + dbeta;
            if (beta >= p[2][2]) break;
            seg_t s;
            if (!segment_ranges(p[0], p[1], p[2], beta, &s)) continue;
            if (stats) stats[1]++;
            /* Step 3: increment the bins of the intersecting circles:
             * 2 on [|C|, min), 1 on [min, max) (G5). */
            for (int c = 0; c < N; ++c) {
                double rho = col_rho(c, R, N) + drho;
                if (s.rc >= 0.0 && s.rc <= rho && rho < s.rmin) img[r * N + c] += 2;
                else if (s.rmin <= rho && rho < s.rmax) img[r * N + c] += 1;
            }
        }
    }
}

/* counts_out: n*N*N exact counts (uint32), row = beta ascending, col = alpha ascending.
 * fragile_out (optional): 1 where the count changes when the circle is moved by
 * tau = tau_rel*R in beta and/or rho: the 8 displacements (a*tau, b*tau), a,b in
 * {-1,0,1}, not both 0.  tau_rel = 1e-5 is the north-star attribution rule ("an
 * intersection within 1e-5 relative of a bin or layer edge"); this is the
 * perturbation reading of DESIGN.md section 2: a pixel whose count is the same at
 * every displacement is NOT fragile even if a decision there is tied (e.g. a
 * circle through an edge shared by two triangles: either triangle counts it).
 * stats (optional, int64[2]): {pairs whose beta-extent meets the image, segments}. */
EXPORT void oracle_rici_generate(const float *vertices, int64_t nv, const int32_t *indices,
                                 int64_t nt, const float *origins, int64_t n, double R, int N,
                                 uint32_t *counts_out, uint8_t *fragile_out, int64_t *stats,
                                 double tau_rel) {
    (void)nv;
    int64_t sp = 0, ss = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : sp, ss)
    for (int64_t i = 0; i < n; ++i) {
        double o[6];
        for (int j = 0; j < 6; ++j) o[j] = origins[6 * i + j];
        frame_t f = spin_frame(o);
        uint32_t *img = counts_out + i * (int64_t)N * N;
        int64_t st[2] = {0, 0};
        image_counts(&f, vertices, indices, nt, R, N, 0.0, 0.0, img, st);
        sp += st[0]; ss += st[1];
        if (fragile_out) {
            uint8_t *fr = fragile_out + i * (int64_t)N * N;
            memset(fr, 0, (size_t)N * N);
            uint32_t *alt = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)N * N);
            const double tau = tau_rel * R;
            for (int a = -1; a <= 1; ++a)
                for (int b = -1; b <= 1; ++b) {
                    if (a == 0 && b == 0) continue;
                    image_counts(&f, vertices, indices, nt, R, N, a * tau, b * tau, alt, NULL);
                    for (int64_t q = 0; q < (int64_t)N * N; ++q)
                        if (alt[q] != img[q]) fr[q] = 1;
                }
            free(alt);
        }
    }
    if (stats) { stats[0] = sp; stats[1] = ss; }
}

/* ------------------------------------------------------------------------ */
/* O-def: the RICI definition itself: pixel (r,c) = number of    */
/* intersections of the circle {(rho_c cos th, rho_c sin th, beta_r)} with   */
/* the surface.  Independent of the paper's algorithm: its own orthonormal   */
/* frame, circle-plane crossing, barycentric inside test.  Exact ties        */
/* (tangency, points on edges) are fragile pixels and are not compared.      */
/* ------------------------------------------------------------------------ */
static void cross3(const double a[3], const double b[3], double o[3]) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
static double dot3(const double a[3], const double b[3]) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

EXPORT void oracle_rici_definition(const float *vertices, int64_t nv, const int32_t *indices,
                                   int64_t nt, const float *origins, int64_t n, double R, int N,
                                   uint32_t *counts_out) {
    (void)nv;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n; ++i) {
        uint32_t *img = counts_out + i * (int64_t)N * N;
        memset(img, 0, sizeof(uint32_t) * (size_t)N * N);
        double s[3] = {origins[6 * i], origins[6 * i + 1], origins[6 * i + 2]};
        double e3[3] = {origins[6 * i + 3], origins[6 * i + 4], origins[6 * i + 5]};
        double l3 = sqrt(dot3(e3, e3));
        if (l3 == 0.0) continue;
        for (int j = 0; j < 3; ++j) e3[j] /= l3;
        double a[3] = {1, 0, 0};
        if (fabs(e3[0]) > 0.9) { a[0] = 0; a[1] = 1; }
        double ad = dot3(a, e3), e1[3], e2[3];
        for (int j = 0; j < 3; ++j) e1[j] = a[j] - ad * e3[j];
        double l1 = sqrt(dot3(e1, e1));
        for (int j = 0; j < 3; ++j) e1[j] /= l1;
        cross3(e3, e1, e2);
        for (int64_t k = 0; k < nt; ++k) {
            double V[3][3];
            for (int j = 0; j < 3; ++j) {
                const float *src = vertices + 3 * (int64_t)indices[3 * k + j];
                double d[3] = {src[0] - s[0], src[1] - s[1], src[2] - s[2]};
                V[j][0] = dot3(d, e1); V[j][1] = dot3(d, e2); V[j][2] = dot3(d, e3);
            }
            double u[3] = {V[1][0] - V[0][0], V[1][1] - V[0][1], V[1][2] - V[0][2]};
            double w[3] = {V[2][0] - V[0][0], V[2][1] - V[0][1], V[2][2] - V[0][2]};
            double m[3];
            cross3(u, w, m);
            if (m[0] == 0.0 && m[1] == 0.0) continue;   /* horizontal / degenerate */
            double dT = dot3(m, V[0]);
            for (int r = 0; r < N; ++r) {
                double beta = row_beta(r, R, N);
                double zmin = fmin(V[0][2], fmin(V[1][2], V[2][2]));
                double zmax = fmax(V[0][2], fmax(V[1][2], V[2][2]));
                if (beta < zmin || beta > zmax) continue;
                for (int c = 0; c < N; ++c) {
                    double rho = col_rho(c, R, N);
                    double A = rho * m[0], B = rho * m[1], C = dT - m[2] * beta;
                    double K = sqrt(A * A + B * B);
                    if (fabs(C) > K) continue;
                    double phi = atan2(B, A), dl = acos(C / K);
                    double th[2] = {phi + dl, phi - dl};
                    int np = (dl == 0.0) ? 1 : 2;
                    for (int q = 0; q < np; ++q) {
                        double X[3] = {rho * cos(th[q]), rho * sin(th[q]), beta};
                        double inside = 1;
                        for (int e = 0; e < 3 && inside; ++e) {
                            const double *P0 = V[e], *P1 = V[(e + 1) % 3];
                            double ed[3] = {P1[0] - P0[0], P1[1] - P0[1], P1[2] - P0[2]};
                            double xd[3] = {X[0] - P0[0], X[1] - P0[1], X[2] - P0[2]};
                            double cr[3];
                            cross3(ed, xd, cr);
                            if (dot3(cr, m) < 0.0) inside = 0;
                        }
                        if (inside) img[r * N + c] += 1;
                    }
                }
            }
        }
    }
}

/* ------------------------------------------------------------------------ */
/* CRSS / CRD: Eq. 6, Eq. 7, Listing 1.      */
/* ------------------------------------------------------------------------ */
/* Index ranges read zero-based: r in [0, N-1], c in [1, N-1] (G7). */
EXPORT uint64_t oracle_crss(const uint16_t *needle, const uint16_t *haystack, int N) {
    int64_t score = 0;
    for (int r = 0; r < N; ++r) {
        for (int c = 1; c < N; ++c) {                   /* "Skip first column" */
            int64_t nd = (int64_t)needle[r * N + c] - (int64_t)needle[r * N + c - 1];
            int64_t hd = (int64_t)haystack[r * N + c] - (int64_t)haystack[r * N + c - 1];
            if (nd != 0) score += (nd - hd) * (nd - hd);
        }
    }
    return (uint64_t)score;
}

EXPORT void oracle_crss_matrix(const uint16_t *needles, int64_t nn, const uint16_t *haystack,
                               int64_t nh, int N, uint64_t *out) {
    const int64_t P = (int64_t)N * N;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < nn; ++i)
        for (int64_t j = 0; j < nh; ++j)
            out[i * nh + j] = oracle_crss(needles + i * P, haystack + j * P, N);
}

/* Rank of needle i's true correspondence (haystack i, G11): the number of
 * haystack images strictly closer than it, so ties take the best rank
 * ("we use the highest (best) rank"; "lower ranks are better"). */
EXPORT void oracle_count_below(const uint16_t *needles, int64_t nn, const uint16_t *haystack,
                               int64_t nh, int N, const uint64_t *thresholds, uint32_t *counts) {
    const int64_t P = (int64_t)N * N;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < nn; ++i) {
        uint32_t cnt = 0;
        for (int64_t j = 0; j < nh; ++j)
            if (oracle_crss(needles + i * P, haystack + j * P, N) < thresholds[i]) cnt++;
        counts[i] = cnt;
    }
}

EXPORT void oracle_ranks(const uint16_t *needles, int64_t nn, const uint16_t *haystack,
                         int64_t nh, int N, uint32_t *ranks) {
    const int64_t P = (int64_t)N * N;
    uint64_t *thr = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(nn > 0 ? nn : 1));
    for (int64_t i = 0; i < nn; ++i) thr[i] = oracle_crss(needles + i * P, haystack + i * P, N);
    oracle_count_below(needles, nn, haystack, nh, N, thr, ranks);
    free(thr);
}

/* ------------------------------------------------------------------------ */
/* Clutter fraction, Eq. 8: clutter = (A_all - A_object) / A_all */
/* where A_all is the surface area of all objects inside the support volume  */
/* and A_object that of the object of interest.  Support volume: the */
/* RICI support cylinder, radius R, beta in [-R/2, R/2] (G4, G17).  The      */
/* paper does not say how the area is measured (G17): each triangle is cut   */
/* into Q*Q congruent sub-triangles (barycentric grid) and a sub-triangle    */
/* counts with area A/Q^2 when its centroid lies inside the volume.          */
/* ------------------------------------------------------------------------ */
static int inside_support(const frame_t *f, const double p[3], double R) {
    double t[3];
    project(f, p, t);
    return fabs(t[2]) <= 0.5 * R && t[0] * t[0] + t[1] * t[1] <= R * R;
}

EXPORT void oracle_clutter_fraction(const float *vertices, int64_t nv, const int32_t *indices, int64_t nt,
                                    const uint8_t *object_tag, const float *origins, int64_t n, double R,
                                    int Q, double *out_fraction, double *out_area_all, double *out_area_obj) {
    (void)nv;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n; ++i) {
        double o[6];
        for (int j = 0; j < 6; ++j) o[j] = origins[6 * i + j];
        frame_t f = spin_frame(o);
        double a_all = 0.0, a_obj = 0.0;
        if (f.valid) {
            for (int64_t k = 0; k < nt; ++k) {
                double v[3][3];
                for (int j = 0; j < 3; ++j)
                    for (int a = 0; a < 3; ++a) v[j][a] = vertices[3 * (int64_t)indices[3 * k + j] + a];
                double e1[3] = {v[1][0] - v[0][0], v[1][1] - v[0][1], v[1][2] - v[0][2]};
                double e2[3] = {v[2][0] - v[0][0], v[2][1] - v[0][1], v[2][2] - v[0][2]};
                double cr[3];
                cross3(e1, e2, cr);
                const double sub = 0.5 * sqrt(dot3(cr, cr)) / ((double)Q * Q);
                double a_in = 0.0;
                for (int u = 0; u < Q; ++u)
                    for (int w = 0; u + w < Q; ++w)
                        for (int up = 0; up < 2; ++up) {
                            if (!up && u + w >= Q - 1) continue;   /* downward sub-triangles */
                            const double bu = (u + (up ? 1.0 / 3.0 : 2.0 / 3.0)) / Q;
                            const double bw = (w + (up ? 1.0 / 3.0 : 2.0 / 3.0)) / Q;
                            double p[3];
                            for (int a = 0; a < 3; ++a) p[a] = v[0][a] + bu * e1[a] + bw * e2[a];
                            if (inside_support(&f, p, R)) a_in += sub;
                        }
                a_all += a_in;
                if (object_tag[k]) a_obj += a_in;
            }
        }
        out_fraction[i] = a_all > 0.0 ? (a_all - a_obj) / a_all : 0.0;
        if (out_area_all) out_area_all[i] = a_all;
        if (out_area_obj) out_area_obj[i] = a_obj;
    }
}

EXPORT int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

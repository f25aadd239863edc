/*
 * morea_oracle.c -- the plain, slow, single-threaded CPU definition of MOREA's
 * data-parallel hot path (arXiv 2303.04873), written from PAPER.md.
 *
 *   *** TEST INFRASTRUCTURE ONLY ***
 *   Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 *   `--impl reference` leg may load or call this library.  It shares no code,
 *   header, table or constant generator with the CUDA path under
 *   paper_2303_04873_b200/, and it includes nothing from there.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (no fast-math, no OpenMP, no
 * SIMD intrinsics) so the fp64 results are reproducible.
 *
 * What it computes (citations are PAPER.md line numbers; readings O1..O13 are
 * listed in DESIGN.md §3 and SURVEY.md §8(c)):
 *   canonical fixed-point coordinates        O1  (paper silent)
 *   signed-volume fold flags + severity      App. A.4, §4.3.1 L431   (O2)
 *   voxel-centre sample sets, exactly-once   App. A.2 L739-742 + north_star   (O3)
 *   piecewise-affine transform T, T'         App. A.2 "barycentric"      (O4)
 *   trilinear interpolation, clamp           App. A.2 L744                    (O5)
 *   h with exact zero/non-zero case split    §4.1.2 eq. L316-323              (O6)
 *   f_intensity                              §4.1.2 eq. L316-317              (O7)
 *   f_guidance, truncated distance maps      §4.1.3 eq. L338-342, App. A.3 L793-796 (O8)
 *   f_magnitude, 10 edges incl. 4 spokes     §4.1.1 eq. L251-259              (O9)
 *   partial evaluation (delta on dependents) §1, §4.2.1 L400-410        (O10)
 *   Sobol-in-tetrahedron sampler (NEXT-1)    App. A.2 L744-751                (S1..S9)
 *   batched fold repair (NEXT-2)             §4.3.1 L429-437                  (P1..P8)
 *   elasticity from masks, DVF (NEXT-4)      App. A.1, §5.4 L616     (E1..E3)
 *   optimal mixing of a colour class (NEXT-3) §3 L231-233                      (M1..M7)
 *
 * Everything that decides an integer (ownership, fold, the h case split, band
 * membership) is decided exactly in integer arithmetic (int64 / __int128) or
 * on identical fp32 values.  Values are fp64.  There is no blocking, fusion or
 * reordering: every sample is visited by a per-voxel loop over each tet's
 * bounding box, exactly as the definitions read.
 *
 * Parity pins for every function live in tests/test_oracle_*.py; the nearest
 * point search used for the distance maps is an exact bucket search pinned to
 * scipy.spatial.cKDTree and to brute force.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

#define ORC_F_DOMAIN 1
#define ORC_F_EMPTY 2
#define ORC_F_COVERAGE 4

/* Q.10 window (O1): Q in [-256*1024, 768*1024) on every axis. */
#define QLO (-256LL * 1024LL)
#define QHI (768LL * 1024LL)

typedef struct {
    double h_sum, g_sum, m_sum, severity;
    int64_t n_samples;
    int32_t folds, flags;
} orc_acc;

/* per-tet record returned by orc_eval_tets: 10 doubles */
enum { PT_H = 0, PT_G, PT_NS, PT_NT, PT_M, PT_FOLD_S, PT_FOLD_T, PT_SEV, PT_DOMAIN, PT_PAD, PT_N };

typedef struct {
    int n[3];
    int64_t V;
    double sp[3];
    float *I[2];
    int K;
    int64_t *coff[2];
    float *cxyz[2];
    double w[2][8 * 0 + 64]; /* pair weights |C_i|/|G| per side (K <= 64) */
    double r;
    int N, T;
    float *base;
    int32_t *tets;
    float *cdelta;
    int spoke_mode;
    signed char *ref;
    /* incidence CSR */
    int32_t *inc_off, *inc;
    /* lazy distance maps: memo[side][pair*V + v]; NaN = unknown, -1 = ">= r, not computed" */
    float *memo[2];
    /* bucket grid for exact nearest-point search */
    int bsz, bn[3];
    int32_t *boff[2][64];
    int32_t *bidx[2][64];
    /* coverage reference (row a9): owned-sample count per side of the base mesh; -1 = unknown */
    int64_t expect[2];
    /* sample set: 0 = exactly-once voxel centres (O3), 1 = Sobol points per tet (NEXT-1) */
    int sampler;
    double rate; /* Sobol samples per voxel of tet volume */
    /* test accessor (orc_sample_map): per-voxel h and fg of the side being sampled */
    double *dump_h;
    uint8_t *dump_fg;
} orc_problem;

/* ------------------------------------------------------------------ */
/* O1: canonical coordinates  Q = round-half-even(1024 B + 1024 O) in fp64 */
/* ------------------------------------------------------------------ */
static int64_t canon(float b, float o) {
    double v = 1024.0 * (double)b + 1024.0 * (double)o;
    return (int64_t)nearbyint(v);
}
static int in_window(const int64_t q[3]) {
    for (int a = 0; a < 3; a++)
        if (q[a] < QLO || q[a] >= QHI) return 0;
    return 1;
}

/* Q[side][k][axis] for the 4 vertices of tet t; returns 0 if any vertex is out of window */
static int tet_coords(const orc_problem *P, const float *off, int t, int64_t Q[2][4][3]) {
    int ok = 1;
    for (int k = 0; k < 4; k++) {
        int j = P->tets[4 * t + k];
        for (int s = 0; s < 2; s++) {
            for (int a = 0; a < 3; a++) {
                float o = off ? off[6 * j + 3 * s + a] : 0.0f;
                Q[s][k][a] = canon(P->base[3 * j + a], o);
            }
            if (!in_window(Q[s][k])) ok = 0;
        }
    }
    return ok;
}

/* signed determinant det[Q1-Q0, Q2-Q0, Q3-Q0] (6 x signed volume, Q units^3), exact */
static i128 det4(const int64_t Q[4][3]) {
    i128 a[3], b[3], c[3];
    for (int i = 0; i < 3; i++) {
        a[i] = Q[1][i] - Q[0][i];
        b[i] = Q[2][i] - Q[0][i];
        c[i] = Q[3][i] - Q[0][i];
    }
    return a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0]) +
           a[2] * (b[0] * c[1] - b[1] * c[0]);
}
static int sgn128(i128 v) { return (v > 0) - (v < 0); }

/* ------------------------------------------------------------------ */
/* O3: inward face normals and the exactly-once ownership predicate     */
/* ------------------------------------------------------------------ */
typedef struct {
    i128 n[4][3];    /* inward normal of the face opposite vertex k */
    int64_t f0[4][3]; /* a vertex on that face */
    i128 absdet;     /* |Delta| */
} tet_faces;

/* returns 0 if the tet is degenerate (Delta = 0): it owns nothing */
static int make_faces(const int64_t Q[4][3], tet_faces *F) {
    i128 d = det4(Q);
    if (d == 0) return 0;
    F->absdet = d < 0 ? -d : d;
    for (int k = 0; k < 4; k++) {
        int f[3], m = 0;
        for (int j = 0; j < 4; j++)
            if (j != k) f[m++] = j;
        i128 u[3], v[3], w[3];
        for (int a = 0; a < 3; a++) {
            u[a] = Q[f[1]][a] - Q[f[0]][a];
            v[a] = Q[f[2]][a] - Q[f[0]][a];
            w[a] = Q[k][a] - Q[f[0]][a];
        }
        i128 n[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
        i128 s = n[0] * w[0] + n[1] * w[1] + n[2] * w[2]; /* = +-Delta */
        for (int a = 0; a < 3; a++) {
            F->n[k][a] = s > 0 ? n[a] : -n[a];
            F->f0[k][a] = Q[f[0]][a];
        }
    }
    return 1;
}

/* e_k(q) = n_k . (1024 q - f0_k): 4 x barycentric numerator, exact */
static i128 face_eval(const tet_faces *F, int k, const int64_t q[3]) {
    i128 e = 0;
    for (int a = 0; a < 3; a++) e += F->n[k][a] * (i128)(1024 * q[a] - F->f0[k][a]);
    return e;
}
/* lexpos(n): first non-zero component positive  (perturbation q + (eps, eps^2, eps^3)) */
static int lexpos(const i128 n[3]) {
    if (n[0] != 0) return n[0] > 0;
    if (n[1] != 0) return n[1] > 0;
    return n[2] > 0;
}
static int owns(const tet_faces *F, const int64_t q[3], i128 e[4]) {
    for (int k = 0; k < 4; k++) {
        e[k] = face_eval(F, k, q);
        if (e[k] > 0) continue;
        if (e[k] == 0 && lexpos(F->n[k])) continue;
        return 0;
    }
    return 1;
}

/* lattice bbox of the tet clipped to the image: ceil(min Q/1024) .. floor(max Q/1024) */
static int64_t floordiv(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q--;
    return q;
}
static int64_t ceildiv(int64_t a, int64_t b) { return -floordiv(-a, b); }
static void tet_bbox(const orc_problem *P, const int64_t Q[4][3], int64_t lo[3], int64_t hi[3]) {
    for (int a = 0; a < 3; a++) {
        int64_t mn = Q[0][a], mx = Q[0][a];
        for (int k = 1; k < 4; k++) {
            if (Q[k][a] < mn) mn = Q[k][a];
            if (Q[k][a] > mx) mx = Q[k][a];
        }
        lo[a] = ceildiv(mn, 1024);
        hi[a] = floordiv(mx, 1024);
        if (lo[a] < 0) lo[a] = 0;
        if (hi[a] > P->n[a] - 1) hi[a] = P->n[a] - 1;
    }
}

static int64_t vidx(const orc_problem *P, int64_t x, int64_t y, int64_t z) {
    return (z * P->n[1] + y) * P->n[0] + x;
}

/* ------------------------------------------------------------------ */
/* O5: trilinear interpolation with clamp to the border (fp64)          */
/* ------------------------------------------------------------------ */
static double trilinear(const orc_problem *P, const float *vol, const double x[3]) {
    int64_t i0[3];
    double f[3];
    for (int a = 0; a < 3; a++) {
        double xc = x[a];
        if (xc < 0.0) xc = 0.0;
        if (xc > (double)(P->n[a] - 1)) xc = (double)(P->n[a] - 1);
        int64_t fl = (int64_t)floor(xc);
        if (fl > P->n[a] - 2) fl = P->n[a] - 2;
        i0[a] = fl;
        f[a] = xc - (double)fl;
    }
    double v = 0.0;
    for (int dz = 0; dz < 2; dz++)
        for (int dy = 0; dy < 2; dy++)
            for (int dx = 0; dx < 2; dx++) {
                double w = (dx ? f[0] : 1.0 - f[0]) * (dy ? f[1] : 1.0 - f[1]) * (dz ? f[2] : 1.0 - f[2]);
                v += w * (double)vol[vidx(P, i0[0] + dx, i0[1] + dy, i0[2] + dz)];
            }
    return v;
}

/* ------------------------------------------------------------------ */
/* O4 + O6: exact transform numerators and the exact contributing set  */
/* ------------------------------------------------------------------ */
/* Position on axis a is x_a = Pnum_a / M with M = 1024 |Delta| > 0 (exact rational).
 * Contributing lattice indices of the clamped trilinear footprint on that axis:
 *   x <= 0      -> {0}
 *   x >= n-1    -> {n-1}
 *   x integer   -> {x}
 *   otherwise   -> {floor x, floor x + 1}                                   */
static int axis_set(i128 Pnum, i128 M, int n, int64_t out[2]) {
    if (Pnum <= 0) { out[0] = 0; return 1; }
    if (Pnum >= (i128)(n - 1) * M) { out[0] = n - 1; return 1; }
    i128 fl = Pnum / M; /* Pnum > 0, M > 0: truncation = floor */
    if (Pnum % M == 0) { out[0] = (int64_t)fl; return 1; }
    out[0] = (int64_t)fl;
    out[1] = (int64_t)fl + 1;
    return 2;
}

/* fg(b): some contributing corner has I > 0 (exactly) */
static int fg_exact(const orc_problem *P, const float *vol, const i128 Pnum[3], i128 M) {
    int64_t s[3][2];
    int c[3];
    for (int a = 0; a < 3; a++) c[a] = axis_set(Pnum[a], M, P->n[a], s[a]);
    for (int k = 0; k < c[2]; k++)
        for (int j = 0; j < c[1]; j++)
            for (int i = 0; i < c[0]; i++)
                if (vol[vidx(P, s[0][i], s[1][j], s[2][k])] > 0.0f) return 1;
    return 0;
}

/* h(a, b) of PAPER.md §4.1.2 L318-322 with the case decided by (a > 0, fg) */
static double h_of(double a, double b, int fg) {
    if (a > 0.0 && fg) return (a - b) * (a - b);
    if (a == 0.0 && !fg) return 0.0;
    return 1.0;
}

/* ------------------------------------------------------------------ */
/* O8: distance maps  D_i(q) = min_c || (q - c) . spacing ||  (fp64 -> fp32) */
/* ------------------------------------------------------------------ */
static double sqdist(const orc_problem *P, const int64_t q[3], const float *c) {
    double dx = ((double)q[0] - (double)c[0]) * P->sp[0];
    double dy = ((double)q[1] - (double)c[1]) * P->sp[1];
    double dz = ((double)q[2] - (double)c[2]) * P->sp[2];
    return dx * dx + dy * dy + dz * dz;
}

static int bucket_of(const orc_problem *P, double c, int a) {
    int b = (int)floor((c + 1.0) / (double)P->bsz);
    if (b < 0) b = 0;
    if (b > P->bn[a] - 1) b = P->bn[a] - 1;
    return b;
}

/* exact min over the pair's points of sqdist, searching buckets in Chebyshev
 * rings around q's bucket; stops only once every unvisited point is provably
 * farther than the best found (or farther than `limit2` if limit2 > 0). */
static double nearest_sq(const orc_problem *P, int side, int pair, const int64_t q[3], double limit2) {
    const float *pts = P->cxyz[side] + 3 * P->coff[side][pair];
    const int32_t *off = P->boff[side][pair];
    const int32_t *idx = P->bidx[side][pair];
    int qb[3];
    for (int a = 0; a < 3; a++) qb[a] = bucket_of(P, (double)q[a], a);
    double smin = P->sp[0];
    if (P->sp[1] < smin) smin = P->sp[1];
    if (P->sp[2] < smin) smin = P->sp[2];
    double best = INFINITY;
    int maxring = P->bn[0];
    if (P->bn[1] > maxring) maxring = P->bn[1];
    if (P->bn[2] > maxring) maxring = P->bn[2];
    for (int ring = 0; ring <= maxring; ring++) {
        for (int bz = qb[2] - ring; bz <= qb[2] + ring; bz++) {
            if (bz < 0 || bz >= P->bn[2]) continue;
            for (int by = qb[1] - ring; by <= qb[1] + ring; by++) {
                if (by < 0 || by >= P->bn[1]) continue;
                for (int bx = qb[0] - ring; bx <= qb[0] + ring; bx++) {
                    if (bx < 0 || bx >= P->bn[0]) continue;
                    int cheb = abs(bx - qb[0]);
                    if (abs(by - qb[1]) > cheb) cheb = abs(by - qb[1]);
                    if (abs(bz - qb[2]) > cheb) cheb = abs(bz - qb[2]);
                    if (cheb != ring) continue;
                    int b = (bz * P->bn[1] + by) * P->bn[0] + bx;
                    for (int32_t t = off[b]; t < off[b + 1]; t++) {
                        double d2 = sqdist(P, q, pts + 3 * idx[t]);
                        if (d2 < best) best = d2;
                    }
                }
            }
        }
        /* any unvisited point lies >= ring*bsz voxels away along some axis
         * (a point at the clamp border can only be farther) */
        double lb = (double)ring * (double)P->bsz * smin;
        double lb2 = lb * lb * (1.0 - 1e-9);
        if (best <= lb2) break;
        if (limit2 > 0.0 && lb2 >= limit2) break;
    }
    return best;
}

/* exact fp32 map value at voxel q for pair i on side s (memoised) */
static float dmap_exact(orc_problem *P, int s, int i, const int64_t q[3]) {
    int64_t v = vidx(P, q[0], q[1], q[2]);
    float *m = &P->memo[s][(int64_t)i * P->V + v];
    if (isnan(*m) || *m < 0.0f) {
        double d2 = nearest_sq(P, s, i, q, 0.0);
        *m = (float)sqrt(d2);
    }
    return *m;
}

/* band membership d = D_i(q) < r; returns 1 and sets *d if in band */
static int band(orc_problem *P, int s, int i, const int64_t q[3], float *d) {
    int64_t v = vidx(P, q[0], q[1], q[2]);
    float *m = &P->memo[s][(int64_t)i * P->V + v];
    if (isnan(*m)) {
        /* any point with sqdist < (r(1+1e-6))^2 ?  if none, D >= r certainly */
        double lim = P->r * (1.0 + 1e-6);
        double d2 = nearest_sq(P, s, i, q, lim * lim);
        if (d2 >= lim * lim) {
            *m = -1.0f; /* marker: >= r, value not needed for the band */
            return 0;
        }
        *m = (float)sqrt(nearest_sq(P, s, i, q, 0.0));
    }
    if (*m < 0.0f) return 0;
    *d = *m;
    return (double)*m < P->r;
}

static double trilinear_map(orc_problem *P, int s, int i, const double x[3]) {
    int64_t i0[3];
    double f[3];
    for (int a = 0; a < 3; a++) {
        double xc = x[a];
        if (xc < 0.0) xc = 0.0;
        if (xc > (double)(P->n[a] - 1)) xc = (double)(P->n[a] - 1);
        int64_t fl = (int64_t)floor(xc);
        if (fl > P->n[a] - 2) fl = P->n[a] - 2;
        i0[a] = fl;
        f[a] = xc - (double)fl;
    }
    double v = 0.0;
    for (int dz = 0; dz < 2; dz++)
        for (int dy = 0; dy < 2; dy++)
            for (int dx = 0; dx < 2; dx++) {
                double w = (dx ? f[0] : 1.0 - f[0]) * (dy ? f[1] : 1.0 - f[1]) * (dz ? f[2] : 1.0 - f[2]);
                int64_t q[3] = {i0[0] + dx, i0[1] + dy, i0[2] + dz};
                v += w * (double)dmap_exact(P, s, i, q);
            }
    return v;
}

/* ------------------------------------------------------------------ */
/* O9: f_magnitude per tet: c_delta * sum over 10 edges (|e_s| - |e_t|)^2, mm */
/* ------------------------------------------------------------------ */
static double edge_len(const orc_problem *P, const int64_t Q[4][3], int kind, int u, int v) {
    double s = 0.0;
    for (int a = 0; a < 3; a++) {
        double comp;
        if (kind == 0) {
            comp = (double)(Q[u][a] - Q[v][a]) / 1024.0;
        } else {
            /* spoke: vertex u -> centroid of the opposite face (SURVEY.md O9 / S:L201),
             * (3 Q_u - sum of the other three) / 3 / 1024; spoke_mode 1 = tet centroid,
             * which is 3/4 of that vector */
            int64_t sum = 0;
            for (int k = 0; k < 4; k++)
                if (k != u) sum += Q[k][a];
            comp = (double)(3 * Q[u][a] - sum) / 3072.0;
            if (P->spoke_mode == 1) comp *= 0.75;
        }
        comp *= P->sp[a];
        s += comp * comp;
    }
    return sqrt(s);
}

static double magnitude(const orc_problem *P, int t, const int64_t Q[2][4][3]) {
    static const int E[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    double m = 0.0;
    for (int e = 0; e < 6; e++) {
        double d = edge_len(P, Q[0], 0, E[e][0], E[e][1]) - edge_len(P, Q[1], 0, E[e][0], E[e][1]);
        m += d * d;
    }
    for (int k = 0; k < 4; k++) {
        double d = edge_len(P, Q[0], 1, k, 0) - edge_len(P, Q[1], 1, k, 0);
        m += d * d;
    }
    return (double)P->cdelta[t] * m;
}

/* ------------------------------------------------------------------ */
/* One tet, one side: visit every lattice point of its bbox, keep the owned */
/* ones, accumulate h (O6/O7) and the guidance term (O8).               */
/* ------------------------------------------------------------------ */
static void tet_side_samples(orc_problem *P, int s, const int64_t Q[2][4][3], double *h_sum,
                             double *g_sum, int64_t *n_owned, int32_t *owner_map, int tet_id) {
    tet_faces F;
    if (!make_faces(Q[s], &F)) return; /* degenerate: owns nothing */
    int so = 1 - s;
    const float *Iown = P->I[s], *Ioth = P->I[so];
    i128 M = (i128)1024 * F.absdet;
    i128 U[4][3];
    for (int k = 0; k < 4; k++)
        for (int a = 0; a < 3; a++) U[k][a] = (i128)(Q[so][k][a] - Q[s][k][a]);
    int64_t lo[3], hi[3];
    tet_bbox(P, Q[s], lo, hi);
    for (int64_t z = lo[2]; z <= hi[2]; z++)
        for (int64_t y = lo[1]; y <= hi[1]; y++)
            for (int64_t x = lo[0]; x <= hi[0]; x++) {
                int64_t q[3] = {x, y, z};
                i128 e[4];
                if (!owns(&F, q, e)) continue;
                if (owner_map) {
                    int64_t v = vidx(P, x, y, z);
                    owner_map[v] = owner_map[v] == -1 ? tet_id : -2;
                    continue;
                }
                (*n_owned)++;
                if (!h_sum) continue; /* count only */
                /* O4: x = q + sum_k lambda_k U_k / 1024, lambda_k = e_k / |Delta| */
                i128 Pnum[3];
                double xp[3];
                for (int a = 0; a < 3; a++) {
                    i128 Nn = 0;
                    for (int k = 0; k < 4; k++) Nn += e[k] * U[k][a];
                    Pnum[a] = (i128)q[a] * M + Nn;
                    xp[a] = (double)q[a] + (double)Nn / ((double)F.absdet * 1024.0);
                }
                double a_val = (double)Iown[vidx(P, x, y, z)];
                double b_val = trilinear(P, Ioth, xp);
                int fg = fg_exact(P, Ioth, Pnum, M);
                *h_sum += h_of(a_val, b_val, fg);
                if (P->dump_h) {
                    P->dump_h[vidx(P, x, y, z)] = h_of(a_val, b_val, fg);
                    P->dump_fg[vidx(P, x, y, z)] = (uint8_t)fg;
                }
                /* O8: guidance over the pairs whose source-side distance is < r */
                for (int i = 0; i < P->K; i++) {
                    float d;
                    if (!band(P, s, i, q, &d)) continue;
                    double Dp = trilinear_map(P, so, i, xp);
                    double dd = (double)d - Dp;
                    *g_sum += P->w[s][i] * ((P->r - (double)d) / P->r) * dd * dd;
                }
            }
}

/* ------------------------------------------------------------------ */
/* NEXT-1: Sobol-in-tetrahedron sampler (App. A.2).            */
/* "We uniformly sample N points in each tetrahedron using its          */
/* barycentric coordinate system, with N being determined by the volume */
/* of the tetrahedron.  For each point, we sample 4 random real numbers */
/* r_i in [0;1] and take -log(r_i) ... normalize the coordinates by     */
/* their sum ... the Sobol sequence ... seeding the Sobol sequence for  */
/* each tetrahedron with a seed derived from its coordinates."          */
/* Readings S1..S9: the point generator (S1-S5) is the   */
/* counter-based generator both implementations write out identically; */
/* everything after it is the method's arithmetic, in fp64 here.        */
/* ------------------------------------------------------------------ */
static uint32_t SOBOL_V[4][32];
static int sobol_ready = 0;

/* S1: direction numbers of the first 4 Sobol dimensions (Joe & Kuo primitive
 * polynomials; dimension 0 is van der Corput).  (s, a, m_1..m_s) per dimension;
 * m_i = 2^s m_{i-s} ^ m_{i-s} ^ XOR_{k=1}^{s-1} 2^k a_k m_{i-k}, v_i = m_i 2^(31-i). */
static void sobol_init(void) {
    static const int S[4] = {0, 1, 2, 3}, A[4] = {0, 0, 1, 1};
    static const uint32_t M0[4][3] = {{0, 0, 0}, {1, 0, 0}, {1, 3, 0}, {1, 3, 1}};
    if (sobol_ready) return;
    for (int j = 0; j < 4; j++) {
        uint64_t m[32];
        int s = S[j];
        for (int i = 0; i < 32; i++) {
            if (s == 0) { m[i] = 1; continue; }
            if (i < s) { m[i] = M0[j][i]; continue; }
            uint64_t v = m[i - s] ^ (m[i - s] << s);
            for (int k = 1; k < s; k++)
                if ((A[j] >> (s - 1 - k)) & 1) v ^= m[i - k] << k;
            m[i] = v;
        }
        for (int i = 0; i < 32; i++) SOBOL_V[j][i] = (uint32_t)(m[i] << (31 - i));
    }
    sobol_ready = 1;
}

/* S2: point k of the sequence in Gray-code order (the order of scipy.stats.qmc.Sobol) */
static void sobol_point(uint64_t k, uint32_t x[4]) {
    uint64_t g = k ^ (k >> 1);
    for (int j = 0; j < 4; j++) {
        uint32_t v = 0;
        for (int b = 0; b < 32; b++)
            if ((g >> b) & 1) v ^= SOBOL_V[j][b];
        x[j] = v;
    }
}

/* S3: seed = FNV-1a (64 bit) over the 12 little-endian int32 Q.10 coordinates of
 * the tet's vertices on the sampled side, in vertex order x, y, z.  S4: the
 * "seeding" is a digital shift: x_j ^ mask_j, mask_j = high 32 bits of
 * splitmix64(seed + j). */
static uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static uint64_t fnv1a64(const unsigned char *b, size_t n) {
    uint64_t h = 14695981039346656037ULL;
    for (size_t i = 0; i < n; i++) {
        h ^= b[i];
        h *= 1099511628211ULL;
    }
    return h;
}
static uint64_t tet_seed(const int64_t Q[4][3]) {
    unsigned char bytes[48];
    for (int k = 0; k < 4; k++)
        for (int a = 0; a < 3; a++) {
            uint32_t c = (uint32_t)(int32_t)Q[k][a];
            for (int b = 0; b < 4; b++) bytes[4 * (3 * k + a) + b] = (unsigned char)((c >> (8 * b)) & 0xFFu);
        }
    return fnv1a64(bytes, 48);
}
static void tet_masks(const int64_t Q[4][3], uint32_t mask[4]) {
    uint64_t seed = tet_seed(Q);
    for (int j = 0; j < 4; j++) mask[j] = (uint32_t)(splitmix64(seed + (uint64_t)j) >> 32);
}

/* S5: r = (x + 1/2) 2^-32 in (0, 1) and -log r (det_ln: log r for r > 0) with a fixed sequence of IEEE
 * double operations (frexp, one division, a degree-23 odd series), so that
 * both implementations get the same bits:  r = m 2^e, m in [sqrt(1/2), sqrt(2)),
 * log m = 2 atanh t, t = (m - 1)/(m + 1), |t| <= 0.1716.  */
static double det_ln(double r) {
    int e;
    double m = frexp(r, &e); /* r = m 2^e, m in [1/2, 1) */
    if (m < 0.70710678118654752440) { m = m * 2.0; e = e - 1; }
    double t = (m - 1.0) / (m + 1.0);
    double t2 = t * t;
    double p = 1.0 / 23.0;
    p = p * t2 + 1.0 / 21.0;
    p = p * t2 + 1.0 / 19.0;
    p = p * t2 + 1.0 / 17.0;
    p = p * t2 + 1.0 / 15.0;
    p = p * t2 + 1.0 / 13.0;
    p = p * t2 + 1.0 / 11.0;
    p = p * t2 + 1.0 / 9.0;
    p = p * t2 + 1.0 / 7.0;
    p = p * t2 + 1.0 / 5.0;
    p = p * t2 + 1.0 / 3.0;
    p = p * t2 + 1.0;
    double lm = 2.0 * t * p;
    /* log 2 = LN2_HI + LN2_LO, LN2_HI with 32 trailing zero bits (e LN2_HI exact) */
    double lr = (double)e * 6.93147180369123816490e-01 + ((double)e * 1.90821492927058770002e-10 + lm);
    return lr;
}
static double neg_log(uint32_t x) {
    double r = ((double)x + 0.5) * 2.3283064365386963e-10; /* 2^-32, exact */
    return -det_ln(r);
}

/* S6: number of samples of a tet side: N = floor(rate |Delta| / (6 1024^3) + 1/2),
 * |Delta| / (6 1024^3) being the volume in voxels (rate 1.0 ~ one sample per voxel) */
static int64_t sobol_count(const orc_problem *P, const int64_t Q[4][3]) {
    i128 d = det4(Q);
    if (d < 0) d = -d;
    double vol = (double)(int64_t)d;
    return (int64_t)floor(vol * (P->rate / 6442450944.0) + 0.5);
}

/* S7: barycentrics lambda_j = e_j / (((e_0 + e_1) + e_2) + e_3), and the point on
 * a side:  X_0 + ((lambda_1 (X_1 - X_0) + lambda_2 (X_2 - X_0)) + lambda_3 (X_3 - X_0)),
 * X = Q / 1024 (exact); the same lambda on both sides (T maps barycentrics). */
static void sobol_lambda(const uint32_t x[4], const uint32_t mask[4], double lam[4]) {
    double e[4];
    for (int j = 0; j < 4; j++) e[j] = neg_log(x[j] ^ mask[j]);
    double s = ((e[0] + e[1]) + e[2]) + e[3];
    for (int j = 0; j < 4; j++) lam[j] = e[j] / s;
}
static void bary_point(const int64_t Q[4][3], const double lam[4], double p[3]) {
    for (int a = 0; a < 3; a++) {
        double x0 = (double)Q[0][a] / 1024.0;
        double d1 = (double)(Q[1][a] - Q[0][a]) / 1024.0;
        double d2 = (double)(Q[2][a] - Q[0][a]) / 1024.0;
        double d3 = (double)(Q[3][a] - Q[0][a]) / 1024.0;
        p[a] = x0 + ((lam[1] * d1 + lam[2] * d2) + lam[3] * d3);
    }
}

/* S8: "value > 0" of the clamped trilinear interpolant at x, decided exactly:
 * some contributing corner (O5/O6 footprint rules on each axis) has I > 0 */
static int positive_at(const orc_problem *P, const float *vol, const double x[3]) {
    int64_t s[3][2];
    int c[3];
    for (int a = 0; a < 3; a++) {
        int n = P->n[a];
        if (x[a] <= 0.0) { s[a][0] = 0; c[a] = 1; continue; }
        if (x[a] >= (double)(n - 1)) { s[a][0] = n - 1; c[a] = 1; continue; }
        double fl = floor(x[a]);
        s[a][0] = (int64_t)fl;
        if (x[a] == fl) { c[a] = 1; continue; }
        s[a][1] = (int64_t)fl + 1;
        c[a] = 2;
    }
    for (int k = 0; k < c[2]; k++)
        for (int j = 0; j < c[1]; j++)
            for (int i = 0; i < c[0]; i++)
                if (vol[vidx(P, s[0][i], s[1][j], s[2][k])] > 0.0f) return 1;
    return 0;
}

/* some corner of the clamped trilinear footprint of x (O5) has D_i^s < r */
static int footprint_touches_band(orc_problem *P, int s, int i, const double x[3]) {
    int64_t i0[3];
    for (int a = 0; a < 3; a++) {
        double xc = x[a];
        if (xc < 0.0) xc = 0.0;
        if (xc > (double)(P->n[a] - 1)) xc = (double)(P->n[a] - 1);
        int64_t fl = (int64_t)floor(xc);
        if (fl > P->n[a] - 2) fl = P->n[a] - 2;
        i0[a] = fl;
    }
    for (int dz = 0; dz < 2; dz++)
        for (int dy = 0; dy < 2; dy++)
            for (int dx = 0; dx < 2; dx++) {
                int64_t q[3] = {i0[0] + dx, i0[1] + dy, i0[2] + dz};
                float d;
                if (band(P, s, i, q, &d)) return 1;
            }
    return 0;
}

/* S9: one tet side in Sobol mode.  a = I_s(p) and b = I_s'(T p) are both trilinear
 * (the paper's "interpolating intensity values between voxel centers", L744);
 * h takes its case from the exact positivity of both; the guidance term uses
 * d = D_i^s(p) (interpolated) for every pair with d < r. */
static void tet_side_sobol(orc_problem *P, int s, const int64_t Q[2][4][3], double *h_sum,
                           double *g_sum, int64_t *n_samples) {
    int so = 1 - s;
    int64_t N = sobol_count(P, Q[s]);
    *n_samples += N;
    uint32_t mask[4];
    tet_masks(Q[s], mask);
    for (int64_t k = 0; k < N; k++) {
        uint32_t x[4];
        double lam[4], p[3], tp[3];
        sobol_point((uint64_t)k, x);
        sobol_lambda(x, mask, lam);
        bary_point(Q[s], lam, p);
        bary_point(Q[so], lam, tp);
        double a = trilinear(P, P->I[s], p);
        double b = trilinear(P, P->I[so], tp);
        int fa = positive_at(P, P->I[s], p), fb = positive_at(P, P->I[so], tp);
        double h = (fa && fb) ? (a - b) * (a - b) : ((!fa && !fb) ? 0.0 : 1.0);
        *h_sum += h;
        for (int i = 0; i < P->K; i++) {
            /* d is a convex combination of the footprint's corner distances: when
             * none of them is < r, d >= r (up to one rounding) and the term is 0,
             * so the exact map values are only needed near the band */
            if (!footprint_touches_band(P, s, i, p)) continue;
            double d = trilinear_map(P, s, i, p);
            if (!(d < P->r)) continue;
            double dd = d - trilinear_map(P, so, i, tp);
            *g_sum += P->w[s][i] * ((P->r - d) / P->r) * dd * dd;
        }
    }
}

/* ------------------------------------------------------------------ */
/* NEXT-2: fold repair (§4.3.1).                      */
/* "For each point in a folded tetrahedron, the method mutates the point */
/* using a Gaussian distribution scaled by its estimated distance to the */
/* surrounding 3D polygon.  After 64 samples, the change with the best   */
/* constraint improvement is selected, if present.  If all samples result */
/* in a deterioration, repair is aborted."  Readings P1..P7. */
/* The Gaussian draws come from a counter-based generator (SplitMix64    */
/* keys, Marsaglia's polar method, det_ln) that both implementations     */
/* write out identically.                                                */
/* ------------------------------------------------------------------ */
#define REPAIR_CANDIDATES 64

/* P5: standard normal pairs for one key: uniforms u, v = (32-bit half + 1/2) 2^-31 - 1
 * (exact), s = u^2 + v^2, rejected unless 0 < s < 1, f = sqrt(-2 ln s / s) */
static void gauss_pair(uint64_t key, uint64_t *ctr, double *z0, double *z1) {
    for (;;) {
        uint64_t w = splitmix64(key + (*ctr)++);
        double u = ((double)(uint32_t)(w >> 32) + 0.5) * 4.656612873077392578125e-10 - 1.0;
        double v = ((double)(uint32_t)w + 0.5) * 4.656612873077392578125e-10 - 1.0;
        double sq = u * u + v * v;
        if (!(sq < 1.0) || sq == 0.0) continue;
        double f = sqrt(-2.0 * det_ln(sq) / sq);
        *z0 = u * f;
        *z1 = v * f;
        return;
    }
}
/* P5: key of candidate c of point j, side s, solution k */
static uint64_t repair_key(uint64_t seed, int64_t k, int s, int j, int c) {
    uint64_t h = splitmix64(seed + (uint64_t)k);
    h = splitmix64(h + (uint64_t)s);
    h = splitmix64(h + (uint64_t)j);
    return splitmix64(h + (uint64_t)c);
}
static void repair_normal3(uint64_t key, double z[3]) {
    uint64_t ctr = 0;
    double d;
    gauss_pair(key, &ctr, &z[0], &z[1]);
    gauss_pair(key, &ctr, &z[2], &d);
}

/* Q of vertex k of tet t on side s, with point j's side-s offset replaced by o3 (if j >= 0) */
static int tet_side_coords(const orc_problem *P, const float *off, int t, int s, int j,
                           const float o3[3], int64_t Q[4][3]) {
    int ok = 1;
    for (int k = 0; k < 4; k++) {
        int v = P->tets[4 * t + k];
        for (int a = 0; a < 3; a++) {
            float o = (v == j) ? o3[a] : off[6 * v + 3 * s + a];
            Q[k][a] = canon(P->base[3 * v + a], o);
        }
        if (!in_window(Q[k])) ok = 0;
    }
    return ok;
}

/* O2 severity of tet t on side s (0 when its sign matches the reference) */
static double side_severity(const orc_problem *P, const int64_t Q[4][3], int t) {
    i128 d = det4(Q);
    if (sgn128(d) == P->ref[t]) return 0.0;
    return (double)(d < 0 ? -d : d) / (6.0 * 1073741824.0) * P->sp[0] * P->sp[1] * P->sp[2];
}

/* P6: constraint score of point j on side s with j's offset o3: (number of folded
 * incident tets, their summed severity), compared lexicographically; a vertex
 * leaving the Q.10 window scores (INT_MAX, +inf) */
typedef struct { int32_t folds; double sev; } repair_score;
static repair_score incident_score(const orc_problem *P, const float *off, int s, int j, const float o3[3]) {
    repair_score r = {0, 0.0};
    for (int32_t u = P->inc_off[j]; u < P->inc_off[j + 1]; u++) {
        int t = P->inc[u];
        int64_t Q[4][3];
        if (!tet_side_coords(P, off, t, s, j, o3, Q)) {
            r.folds = 0x7fffffff;
            r.sev = INFINITY;
            return r;
        }
        if (sgn128(det4(Q)) != P->ref[t]) {
            r.folds++;
            r.sev += side_severity(P, Q, t);
        }
    }
    return r;
}
static int score_less(repair_score a, repair_score b) {
    return a.folds < b.folds || (a.folds == b.folds && a.sev < b.sev);
}

/* P4: sigma = 1/2 min over the incident tets (unfolded ones, else all) of the distance
 * from j to the plane of its opposite face, |Delta| / (1024 |n|), voxel units; 1/2 if none */
static double repair_sigma(const orc_problem *P, const float *off, int s, int j) {
    double best[2] = {INFINITY, INFINITY}; /* [unfolded only, all] */
    for (int32_t u = P->inc_off[j]; u < P->inc_off[j + 1]; u++) {
        int t = P->inc[u];
        int64_t Q[4][3];
        if (!tet_side_coords(P, off, t, s, -1, NULL, Q)) continue;
        int kj = 0;
        for (int k = 0; k < 4; k++)
            if (P->tets[4 * t + k] == j) kj = k;
        int f[3], m = 0;
        for (int k = 0; k < 4; k++)
            if (k != kj) f[m++] = k;
        double e1[3], e2[3];
        for (int a = 0; a < 3; a++) {
            e1[a] = (double)(Q[f[1]][a] - Q[f[0]][a]);
            e2[a] = (double)(Q[f[2]][a] - Q[f[0]][a]);
        }
        double n0 = e1[1] * e2[2] - e1[2] * e2[1];
        double n1 = e1[2] * e2[0] - e1[0] * e2[2];
        double n2 = e1[0] * e2[1] - e1[1] * e2[0];
        double nn = sqrt(n0 * n0 + n1 * n1 + n2 * n2);
        if (!(nn > 0.0)) continue;
        i128 d = det4(Q);
        double dist = (double)(int64_t)(d < 0 ? -d : d) / (nn * 1024.0);
        if (dist < best[1]) best[1] = dist;
        if (sgn128(d) == P->ref[t] && dist < best[0]) best[0] = dist;
    }
    double b = best[0] < INFINITY ? best[0] : best[1];
    return b < INFINITY ? 0.5 * b : 0.5;
}

/* P1-P8 for one solution (index k for the generator); offsets updated in place.
 * fixed: NULL or N*3 flags of axes the repair must not move (P8, e.g. hull points
 * constrained to their boundary planes, fixed corners); they apply to both sides. */
int orc_repair(orc_problem *P, float *off, const uint8_t *fixed, uint64_t seed, int64_t k,
               int32_t *moved, int32_t *aborted) {
    *moved = *aborted = 0;
    char *pts = (char *)malloc(P->N);
    for (int s = 0; s < 2; s++) {
        /* P1/P2: vertices of the tets folded on side s at the start of the pass */
        memset(pts, 0, P->N);
        for (int t = 0; t < P->T; t++) {
            int64_t Q[4][3];
            if (!tet_side_coords(P, off, t, s, -1, NULL, Q)) continue;
            if (sgn128(det4(Q)) != P->ref[t])
                for (int v = 0; v < 4; v++) pts[P->tets[4 * t + v]] = 1;
        }
        for (int j = 0; j < P->N; j++) {
            if (!pts[j]) continue;
            float cur[3];
            for (int a = 0; a < 3; a++) cur[a] = off[6 * j + 3 * s + a];
            repair_score s0 = incident_score(P, off, s, j, cur);
            /* P3: no folded incident tet left (earlier moves fixed them): nothing to do */
            if (s0.folds == 0) continue;
            double sigma = repair_sigma(P, off, s, j);
            repair_score best = {0x7fffffff, INFINITY};
            int best_c = -1;
            float best_o[3] = {0, 0, 0};
            for (int c = 0; c < REPAIR_CANDIDATES; c++) {
                double z[3];
                repair_normal3(repair_key(seed, k, s, j, c), z);
                float o3[3];
                for (int a = 0; a < 3; a++)
                    o3[a] = (fixed && fixed[3 * j + a]) ? cur[a] : (float)((double)cur[a] + sigma * z[a]);
                repair_score sc = incident_score(P, off, s, j, o3);
                if (score_less(sc, best)) { /* strict: the lowest index wins ties */
                    best = sc;
                    best_c = c;
                    for (int a = 0; a < 3; a++) best_o[a] = o3[a];
                }
            }
            /* P7: apply the best candidate if it strictly improves, else abort the point */
            if (best_c >= 0 && score_less(best, s0)) {
                for (int a = 0; a < 3; a++) off[6 * j + 3 * s + a] = best_o[a];
                (*moved)++;
            } else {
                (*aborted)++;
            }
        }
    }
    free(pts);
    return 0;
}

/* per-tet contributions (both sides) for one solution */
static void tet_contrib(orc_problem *P, const float *off, int t, double rec[PT_N]) {
    memset(rec, 0, sizeof(double) * PT_N);
    int64_t Q[2][4][3];
    if (!tet_coords(P, off, t, Q)) {
        rec[PT_DOMAIN] = 1.0;
        return;
    }
    for (int s = 0; s < 2; s++) {
        i128 d = det4(Q[s]);
        if (sgn128(d) != P->ref[t]) { /* O2: sign change, zero counts as a fold */
            rec[s == 0 ? PT_FOLD_S : PT_FOLD_T] = 1.0;
            double vol = (double)(d < 0 ? -d : d) / (6.0 * 1073741824.0);
            rec[PT_SEV] += vol * P->sp[0] * P->sp[1] * P->sp[2];
        }
        int64_t n = 0;
        if (P->sampler == 1) tet_side_sobol(P, s, Q, &rec[PT_H], &rec[PT_G], &n);
        else tet_side_samples(P, s, Q, &rec[PT_H], &rec[PT_G], &n, NULL, t);
        rec[s == 0 ? PT_NS : PT_NT] = (double)n;
    }
    rec[PT_M] = magnitude(P, t, Q);
}

/* ------------------------------------------------------------------ */
/* Public entry points (ctypes)                                        */
/* ------------------------------------------------------------------ */
void orc_destroy(orc_problem *P);

orc_problem *orc_create(int nx, int ny, int nz, const double *spacing, const float *I_s,
                        const float *I_t, int K, const int64_t *cs_off, const float *cs_xyz,
                        const int64_t *ct_off, const float *ct_xyz, double r_mm, int N,
                        const float *base, int T, const int32_t *tets, const float *c_delta,
                        int spoke_mode, int *status) {
    *status = 0;
    if (nx < 2 || ny < 2 || nz < 2 || K < 0 || K > 64 || N < 4 || T < 1) { *status = -1; return NULL; }
    orc_problem *P = (orc_problem *)calloc(1, sizeof(orc_problem));
    P->n[0] = nx; P->n[1] = ny; P->n[2] = nz;
    P->V = (int64_t)nx * ny * nz;
    for (int a = 0; a < 3; a++) P->sp[a] = spacing[a];
    const float *Is[2] = {I_s, I_t};
    const int64_t *co[2] = {cs_off, ct_off};
    const float *cx[2] = {cs_xyz, ct_xyz};
    for (int s = 0; s < 2; s++) {
        P->I[s] = (float *)malloc(sizeof(float) * P->V);
        memcpy(P->I[s], Is[s], sizeof(float) * P->V);
        P->coff[s] = (int64_t *)malloc(sizeof(int64_t) * (K + 1));
        memcpy(P->coff[s], co[s], sizeof(int64_t) * (K + 1));
        int64_t M = co[s][K];
        P->cxyz[s] = (float *)malloc(sizeof(float) * 3 * (M > 0 ? M : 1));
        if (M > 0) memcpy(P->cxyz[s], cx[s], sizeof(float) * 3 * M);
        /* w_i = |C_i| / |G_side| */
        for (int i = 0; i < K; i++) P->w[s][i] = M > 0 ? (double)(co[s][i + 1] - co[s][i]) / (double)M : 0.0;
        P->memo[s] = (float *)malloc(sizeof(float) * P->V * (K > 0 ? K : 1));
        for (int64_t v = 0; v < P->V * (K > 0 ? K : 1); v++) P->memo[s][v] = NAN;
    }
    P->K = K;
    /* r = 2.5 % of the image width (App. A.3) when not given */
    P->r = r_mm > 0.0 ? r_mm : 0.025 * (double)nx * spacing[0];
    P->N = N;
    P->T = T;
    P->base = (float *)malloc(sizeof(float) * 3 * N);
    memcpy(P->base, base, sizeof(float) * 3 * N);
    P->tets = (int32_t *)malloc(sizeof(int32_t) * 4 * T);
    memcpy(P->tets, tets, sizeof(int32_t) * 4 * T);
    P->cdelta = (float *)malloc(sizeof(float) * T);
    for (int t = 0; t < T; t++) P->cdelta[t] = c_delta ? c_delta[t] : 1.0f;
    P->spoke_mode = spoke_mode;
    P->ref = (signed char *)malloc(T);
    for (int t = 0; t < 4 * T; t++)
        if (tets[t] < 0 || tets[t] >= N) { *status = -1; orc_destroy(P); return NULL; }
    /* reference signs from the initial mesh (App. A.4) */
    for (int t = 0; t < T; t++) {
        int64_t Q[2][4][3];
        if (!tet_coords(P, NULL, t, Q)) { *status = -3; orc_destroy(P); return NULL; }
        int sg = sgn128(det4(Q[0]));
        if (sg == 0) { *status = -3; orc_destroy(P); return NULL; }
        P->ref[t] = (signed char)sg;
    }
    /* incidence CSR: tets incident to each point */
    P->inc_off = (int32_t *)calloc(N + 1, sizeof(int32_t));
    for (int t = 0; t < 4 * T; t++) P->inc_off[tets[t] + 1]++;
    for (int j = 0; j < N; j++) P->inc_off[j + 1] += P->inc_off[j];
    P->inc = (int32_t *)malloc(sizeof(int32_t) * 4 * T);
    int32_t *fill = (int32_t *)calloc(N, sizeof(int32_t));
    for (int t = 0; t < T; t++)
        for (int k = 0; k < 4; k++) {
            int j = tets[4 * t + k];
            int dup = 0;
            for (int32_t u = P->inc_off[j]; u < P->inc_off[j] + fill[j]; u++)
                if (P->inc[u] == t) dup = 1;
            if (!dup) P->inc[P->inc_off[j] + fill[j]++] = t;
        }
    /* compact (a tet listing a point twice is invalid anyway) */
    free(fill);
    /* bucket grid for the nearest-point search */
    P->expect[0] = P->expect[1] = -1;
    P->sampler = 0;
    P->rate = 1.0;
    sobol_init();
    P->bsz = 4;
    for (int a = 0; a < 3; a++) P->bn[a] = (P->n[a] + 2) / P->bsz + 1;
    int nb = P->bn[0] * P->bn[1] * P->bn[2];
    for (int s = 0; s < 2; s++)
        for (int i = 0; i < K; i++) {
            int64_t c0 = P->coff[s][i], c1 = P->coff[s][i + 1];
            int32_t *off = (int32_t *)calloc(nb + 1, sizeof(int32_t));
            int32_t *idx = (int32_t *)malloc(sizeof(int32_t) * (c1 - c0 + 1));
            int *bid = (int *)malloc(sizeof(int) * (c1 - c0 + 1));
            for (int64_t c = c0; c < c1; c++) {
                const float *p = P->cxyz[s] + 3 * c;
                int b = (bucket_of(P, p[2], 2) * P->bn[1] + bucket_of(P, p[1], 1)) * P->bn[0] +
                        bucket_of(P, p[0], 0);
                bid[c - c0] = b;
                off[b + 1]++;
            }
            for (int b = 0; b < nb; b++) off[b + 1] += off[b];
            int32_t *cur = (int32_t *)malloc(sizeof(int32_t) * (nb + 1));
            memcpy(cur, off, sizeof(int32_t) * (nb + 1));
            for (int64_t c = c0; c < c1; c++) idx[cur[bid[c - c0]]++] = (int32_t)(c - c0);
            free(cur);
            free(bid);
            P->boff[s][i] = off;
            P->bidx[s][i] = idx;
        }
    return P;
}

void orc_destroy(orc_problem *P) {
    if (!P) return;
    for (int s = 0; s < 2; s++) {
        free(P->I[s]); free(P->coff[s]); free(P->cxyz[s]); free(P->memo[s]);
        for (int i = 0; i < 64; i++) { free(P->boff[s][i]); free(P->bidx[s][i]); }
    }
    free(P->base); free(P->tets); free(P->cdelta); free(P->ref); free(P->inc_off); free(P->inc);
    free(P);
}

/* per-tet records (PT_N doubles each) for the tets in `sub` (or all when sub == NULL) */
int orc_eval_tets(orc_problem *P, const float *offsets_one, int n_sub, const int32_t *sub, double *out) {
    int n = sub ? n_sub : P->T;
    for (int i = 0; i < n; i++) tet_contrib(P, offsets_one, sub ? sub[i] : i, out + (int64_t)PT_N * i);
    return 0;
}

static void acc_objectives(const orc_problem *P, const orc_acc *acc, double obj[3]) {
    if ((acc->flags & (ORC_F_DOMAIN | ORC_F_EMPTY)) || acc->n_samples == 0) {
        obj[0] = obj[1] = obj[2] = NAN;
        return;
    }
    obj[0] = acc->m_sum / (10.0 * (double)P->T);          /* L258 */
    obj[1] = acc->h_sum / (double)acc->n_samples;          /* L317 */
    obj[2] = acc->g_sum / (double)acc->n_samples;          /* L339 */
}

static int any_out_of_window(const orc_problem *P, const float *off) {
    for (int j = 0; j < P->N; j++)
        for (int s = 0; s < 2; s++) {
            int64_t q[3];
            for (int a = 0; a < 3; a++) q[a] = canon(P->base[3 * j + a], off[6 * j + 3 * s + a]);
            if (!in_window(q)) return 1;
        }
    return 0;
}

/* coverage reference: owned voxel centres per side at the base mesh (zero offsets) */
static void base_counts(orc_problem *P) {
    if (P->expect[0] >= 0) return;
    int64_t c[2] = {0, 0};
    for (int t = 0; t < P->T; t++) {
        int64_t Q[2][4][3];
        if (!tet_coords(P, NULL, t, Q)) continue;
        for (int s = 0; s < 2; s++) tet_side_samples(P, s, Q, NULL, NULL, &c[s], NULL, t);
    }
    P->expect[0] = c[0];
    P->expect[1] = c[1];
}

/* full evaluation of one solution (sum over all tets in index order) */
int orc_eval(orc_problem *P, const float *offsets_one, double obj[3], orc_acc *acc) {
    memset(acc, 0, sizeof(*acc));
    double rec[PT_N];
    int64_t ns = 0, nt = 0;
    if (P->sampler == 0) base_counts(P);
    for (int t = 0; t < P->T; t++) {
        tet_contrib(P, offsets_one, t, rec);
        ns += (int64_t)rec[PT_NS];
        nt += (int64_t)rec[PT_NT];
        acc->h_sum += rec[PT_H];
        acc->g_sum += rec[PT_G];
        acc->m_sum += rec[PT_M];
        acc->severity += rec[PT_SEV];
        acc->n_samples += (int64_t)rec[PT_NS] + (int64_t)rec[PT_NT];
        acc->folds += (int32_t)rec[PT_FOLD_S] + (int32_t)rec[PT_FOLD_T];
    }
    if (any_out_of_window(P, offsets_one)) acc->flags |= ORC_F_DOMAIN;
    else if (P->sampler == 0 && (ns != P->expect[0] || nt != P->expect[1]))
        acc->flags |= ORC_F_COVERAGE; /* a9 */
    if (acc->n_samples == 0) acc->flags |= ORC_F_EMPTY;
    acc_objectives(P, acc, obj);
    return 0;
}

/* O10: partial evaluation of one group S for one solution.
 * D = union of the tets incident to S; acc' = acc - sum_D old + sum_D new. */
int orc_eval_partial(orc_problem *P, const float *base_offsets_one, const orc_acc *base_acc,
                     int n_changed, const int32_t *changed, const float *new_vals, double obj[3],
                     orc_acc *acc) {
    char *in_d = (char *)calloc(P->T, 1);
    for (int i = 0; i < n_changed; i++) {
        int j = changed[i];
        if (j < 0 || j >= P->N) { free(in_d); return -1; }
        for (int32_t u = P->inc_off[j]; u < P->inc_off[j + 1]; u++) in_d[P->inc[u]] = 1;
    }
    float *nw = (float *)malloc(sizeof(float) * 6 * P->N);
    memcpy(nw, base_offsets_one, sizeof(float) * 6 * P->N);
    for (int i = 0; i < n_changed; i++)
        for (int c = 0; c < 6; c++) nw[6 * changed[i] + c] = new_vals[6 * i + c];
    *acc = *base_acc;
    double ro[PT_N], rn[PT_N];
    int dom_new = 0;
    for (int t = 0; t < P->T; t++) {
        if (!in_d[t]) continue;
        tet_contrib(P, base_offsets_one, t, ro);
        tet_contrib(P, nw, t, rn);
        acc->h_sum += rn[PT_H] - ro[PT_H];
        acc->g_sum += rn[PT_G] - ro[PT_G];
        acc->m_sum += rn[PT_M] - ro[PT_M];
        acc->severity += rn[PT_SEV] - ro[PT_SEV];
        acc->n_samples += (int64_t)(rn[PT_NS] + rn[PT_NT]) - (int64_t)(ro[PT_NS] + ro[PT_NT]);
        acc->folds += (int32_t)(rn[PT_FOLD_S] + rn[PT_FOLD_T]) - (int32_t)(ro[PT_FOLD_S] + ro[PT_FOLD_T]);
        if (rn[PT_DOMAIN] != 0.0) dom_new = 1;
    }
    acc->flags = (base_acc->flags & ORC_F_DOMAIN) | (dom_new ? ORC_F_DOMAIN : 0);
    for (int i = 0; i < n_changed; i++)
        for (int s = 0; s < 2; s++) {
            int64_t q[3];
            for (int a = 0; a < 3; a++) q[a] = canon(P->base[3 * changed[i] + a], new_vals[6 * i + 3 * s + a]);
            if (!in_window(q)) acc->flags |= ORC_F_DOMAIN;
        }
    if (acc->n_samples == 0) acc->flags |= ORC_F_EMPTY;
    acc_objectives(P, acc, obj);
    free(in_d);
    free(nw);
    return 0;
}

/* ------------------------------------------------------------------ */
/* NEXT-3: optimal mixing of one FOS colour class (§3).        */
/* "Variation then proceeds by considering variables in FOS elements    */
/* jointly in a procedure called optimal mixing.  In this step,         */
/* distributions are estimated for each FOS element in each cluster, and */
/* new, partial solutions are sampled from these distributions.  Newly  */
/* sampled partial solutions are evaluated and accepted if their        */
/* insertion into the parent solution results in a solution that        */
/* dominates the parent solution or that is non-dominated in the current */
/* elitist archive."  Readings M1..M7.  The distributions   */
/* (mean, Cholesky factor) are inputs: estimating them is the caller's.  */
/* ------------------------------------------------------------------ */
static uint64_t mix_key(uint64_t seed, int64_t gen, int64_t k, int g) {
    uint64_t h = splitmix64(seed + (uint64_t)gen);
    h = splitmix64(h + (uint64_t)k);
    return splitmix64(h + (uint64_t)g);
}

/* a dominates b: no worse in every objective, better in one (minimisation) */
static int dominates(const double a[3], const double b[3]) {
    int better = 0;
    for (int i = 0; i < 3; i++) {
        if (a[i] > b[i]) return 0;
        if (a[i] < b[i]) better = 1;
    }
    return better;
}

/* M1-M7 for one solution (global index k, model of its cluster: mu = sum_g d_g
 * doubles, L = sum_g d_g^2 doubles, row-major lower triangles, d_g = 6 |S_g|);
 * off, acc and obj are updated in place; accepted: G flags */
int orc_mix(orc_problem *P, float *off, orc_acc *acc, double obj[3], int G, const int32_t *grp_off,
            const int32_t *changed, const double *mu, const double *L, const uint8_t *fixed, int A,
            const double *archive, double steer_max, uint64_t seed, int64_t gen, int64_t k,
            uint8_t *accepted) {
    int64_t mo = 0, lo = 0;
    for (int g = 0; g < G; g++) {
        int ns = grp_off[g + 1] - grp_off[g];
        int d = 6 * ns;
        const int32_t *S = changed + grp_off[g];
        accepted[g] = 0;
        /* M1: z ~ N(0, I_d), pairs from the P5 generator keyed by (seed, gen, k, g) */
        double *z = (double *)malloc(sizeof(double) * (d + 1));
        uint64_t key = mix_key(seed, gen, k, g), ctr = 0;
        for (int i = 0; i < d; i += 2) gauss_pair(key, &ctr, &z[i], &z[i + 1]);
        /* M2/M3: x = mu + L z (ascending j), rounded to fp32; fixed axes keep the parent */
        float *nv = (float *)malloc(sizeof(float) * (d > 0 ? d : 1));
        for (int i = 0; i < d; i++) {
            double x = mu[mo + i];
            for (int j = 0; j <= i; j++) x = x + L[lo + (int64_t)i * d + j] * z[j];
            int pt = S[i / 6], c = i % 6;
            nv[i] = (fixed && fixed[3 * pt + c % 3]) ? off[6 * pt + c] : (float)x;
        }
        mo += d;
        lo += (int64_t)d * d;
        /* partial evaluation of the candidate against the current parent */
        double cobj[3];
        orc_acc cacc;
        int rc = orc_eval_partial(P, off, acc, ns, S, nv, cobj, &cacc);
        int ok = rc == 0 && cacc.folds == 0 && !(cacc.flags & (ORC_F_DOMAIN | ORC_F_EMPTY)); /* M4 */
        if (ok && steer_max > 0.0 && !(cobj[2] <= steer_max)) ok = 0;                       /* M5 */
        if (ok) {                                                                             /* M5 */
            int acc_ok = dominates(cobj, obj);
            if (!acc_ok) {
                acc_ok = 1;
                for (int a = 0; a < A; a++)
                    if (dominates(archive + 3 * a, cobj)) { acc_ok = 0; break; }
            }
            ok = acc_ok;
        }
        if (ok) { /* M6: commit; the next group sees the updated parent */
            for (int i = 0; i < ns; i++)
                for (int c = 0; c < 6; c++) off[6 * S[i] + c] = nv[6 * i + c];
            *acc = cacc;
            for (int i = 0; i < 3; i++) obj[i] = cobj[i];
            accepted[g] = 1;
        }
        free(z);
        free(nv);
    }
    return 0;
}

/* fold flags per (side, tet) + count and severity (O2; row a9) */
int orc_check_folds(orc_problem *P, const float *offsets_one, int32_t *count, double *severity,
                    uint8_t *flags /* 2*T or NULL */) {
    *count = 0;
    *severity = 0.0;
    for (int t = 0; t < P->T; t++) {
        int64_t Q[2][4][3];
        if (!tet_coords(P, offsets_one, t, Q)) {
            if (flags) flags[t] = flags[P->T + t] = 0;
            continue;
        }
        for (int s = 0; s < 2; s++) {
            i128 d = det4(Q[s]);
            int f = sgn128(d) != P->ref[t];
            if (flags) flags[(int64_t)s * P->T + t] = (uint8_t)f;
            if (f) {
                (*count)++;
                *severity += (double)(d < 0 ? -d : d) / (6.0 * 1073741824.0) * P->sp[0] * P->sp[1] * P->sp[2];
            }
        }
    }
    return 0;
}

/* test accessor: h and fg (the exact O6 case decision) of every voxel centre
 * sampled on `side` for one solution (fg 255 / h NaN where no tet owns it);
 * the same per-sample arithmetic as orc_eval, written out per voxel. */
int orc_sample_map(orc_problem *P, const float *offsets_one, int side, double *h, uint8_t *fg) {
    for (int64_t v = 0; v < P->V; v++) {
        h[v] = NAN;
        fg[v] = 255;
    }
    P->dump_h = h;
    P->dump_fg = fg;
    for (int t = 0; t < P->T; t++) {
        int64_t Q[2][4][3];
        if (!tet_coords(P, offsets_one, t, Q)) continue;
        double hs = 0.0, gs = 0.0;
        int64_t n = 0;
        tet_side_samples(P, side, Q, &hs, &gs, &n, NULL, t);
    }
    P->dump_h = NULL;
    P->dump_fg = NULL;
    return 0;
}

/* owner of every voxel on one side: tet id, -1 none, -2 more than one (O3) */
int orc_owner_map(orc_problem *P, const float *offsets_one, int side, int32_t *owner) {
    for (int64_t v = 0; v < P->V; v++) owner[v] = -1;
    for (int t = 0; t < P->T; t++) {
        int64_t Q[2][4][3];
        if (!tet_coords(P, offsets_one, t, Q)) continue;
        tet_side_samples(P, side, Q, NULL, NULL, NULL, owner, t);
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* NEXT-4: rasterizer reuse (App. A.1; §5.4).  Readings    */
/* E1..E3.                                                   */
/* ------------------------------------------------------------------ */
/* E1: label of a voxel from an object bitmask byte: 1 + index of the lowest set
 * bit below M (objects in priority order), 0 = no object */
static int voxel_label(uint8_t m, int M) {
    for (int b = 0; b < M; b++)
        if ((m >> b) & 1) return b + 1;
    return 0;
}

/* E1: per tet, the number of owned voxel centres (O3) of each label on side s;
 * counts: T*(M+1), offsets NULL = the base mesh */
int orc_label_counts(orc_problem *P, const float *offsets_one, int s, const uint8_t *masks, int M,
                     int64_t *counts) {
    if (M < 0 || M > 8) return -1;
    memset(counts, 0, sizeof(int64_t) * (size_t)P->T * (M + 1));
    for (int t = 0; t < P->T; t++) {
        int64_t Q[2][4][3];
        if (!tet_coords(P, offsets_one, t, Q)) continue;
        tet_faces F;
        if (!make_faces(Q[s], &F)) continue;
        int64_t lo[3], hi[3];
        tet_bbox(P, Q[s], lo, hi);
        for (int64_t z = lo[2]; z <= hi[2]; z++)
            for (int64_t y = lo[1]; y <= hi[1]; y++)
                for (int64_t x = lo[0]; x <= hi[0]; x++) {
                    int64_t q[3] = {x, y, z};
                    i128 e[4];
                    if (!owns(&F, q, e)) continue;
                    counts[(int64_t)t * (M + 1) + voxel_label(masks[vidx(P, x, y, z)], M)]++;
                }
    }
    return 0;
}

/* E2: c_delta = mean over the tet's owned source voxels (base mesh) of the factor of
 * their label (1.0 for no object): = sum_m frac_m f_m + (1 - sum_m frac_m) 1.0
 * (App. A.1); 1.0 for a tet that owns no voxel */
int orc_elasticity(orc_problem *P, const uint8_t *masks, int M, const float *factors, float *c_out) {
    int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)P->T * (M + 1));
    int rc = orc_label_counts(P, NULL, 0, masks, M, cnt);
    if (rc) { free(cnt); return rc; }
    for (int t = 0; t < P->T; t++) {
        int64_t tot = 0;
        double acc = 0.0;
        for (int b = 0; b <= M; b++) {
            int64_t c = cnt[(int64_t)t * (M + 1) + b];
            tot += c;
            acc += (double)c * (b == 0 ? 1.0 : (double)factors[b - 1]);
        }
        c_out[t] = tot > 0 ? (float)(acc / (double)tot) : 1.0f;
    }
    free(cnt);
    return 0;
}

/* E3: deformation vector field of side s: at every voxel centre q owned on side s,
 * T(q) - q in mm (O4 transform, exact numerator, one fp64 rounding, then x spacing,
 * rounded to fp32); the owner is the lowest tet id when a fold makes several;
 * uncovered voxels get 0 and cov = 0 */
int orc_dvf(orc_problem *P, const float *offsets_one, int s, float *dvf, uint8_t *cov) {
    int32_t *own = (int32_t *)malloc(sizeof(int32_t) * P->V);
    for (int64_t v = 0; v < P->V; v++) own[v] = -1;
    memset(dvf, 0, sizeof(float) * 3 * P->V);
    if (cov) memset(cov, 0, P->V);
    for (int pass = 0; pass < 2; pass++)
        for (int t = 0; t < P->T; t++) {
            int64_t Q[2][4][3];
            if (!tet_coords(P, offsets_one, t, Q)) continue;
            tet_faces F;
            if (!make_faces(Q[s], &F)) continue;
            int so = 1 - s;
            i128 U[4][3];
            for (int k = 0; k < 4; k++)
                for (int a = 0; a < 3; a++) U[k][a] = (i128)(Q[so][k][a] - Q[s][k][a]);
            int64_t lo[3], hi[3];
            tet_bbox(P, Q[s], lo, hi);
            for (int64_t z = lo[2]; z <= hi[2]; z++)
                for (int64_t y = lo[1]; y <= hi[1]; y++)
                    for (int64_t x = lo[0]; x <= hi[0]; x++) {
                        int64_t q[3] = {x, y, z};
                        i128 e[4];
                        if (!owns(&F, q, e)) continue;
                        int64_t v = vidx(P, x, y, z);
                        if (pass == 0) {
                            if (own[v] == -1 || t < own[v]) own[v] = t;
                            continue;
                        }
                        if (own[v] != t) continue;
                        for (int a = 0; a < 3; a++) {
                            i128 Nn = 0;
                            for (int k = 0; k < 4; k++) Nn += e[k] * U[k][a];
                            double u = (double)Nn / ((double)F.absdet * 1024.0);
                            dvf[3 * v + a] = (float)(u * P->sp[a]);
                        }
                        if (cov) cov[v] = 1;
                    }
        }
    free(own);
    return 0;
}

/* full fp32 distance map of pair i on side s (exact nearest-point distances) */
int orc_distance_map(orc_problem *P, int s, int i, float *out) {
    for (int64_t z = 0; z < P->n[2]; z++)
        for (int64_t y = 0; y < P->n[1]; y++)
            for (int64_t x = 0; x < P->n[0]; x++) {
                int64_t q[3] = {x, y, z};
                out[vidx(P, x, y, z)] = dmap_exact(P, s, i, q);
            }
    return 0;
}

/* D_i^s at n given voxel centres q (n x 3, voxel indices): the same exact value
 * the maps above hold (test access for large configs, no new arithmetic). */
int orc_distance_at(orc_problem *P, int s, int i, int64_t n, const int64_t *q, float *out) {
    for (int64_t k = 0; k < n; k++) out[k] = dmap_exact(P, s, i, q + 3 * k);
    return 0;
}

/* debug: one sample of tet t on side s at lattice point q.
 * out = {owned, x, y, z (fp64 transformed position), a, b, fg, h,
 *        floor/integer code per axis (3 values: 2*set_size + (first index sign))} */
int orc_sample_debug(orc_problem *P, const float *offsets_one, int t, int s, const int64_t *q,
                     double *out, int64_t *sets /* 3 x 3: count, idx0, idx1 */) {
    int64_t Q[2][4][3];
    memset(out, 0, sizeof(double) * 8);
    if (!tet_coords(P, offsets_one, t, Q)) return -1;
    tet_faces F;
    if (!make_faces(Q[s], &F)) return -2;
    i128 e[4];
    int o = owns(&F, q, e);
    out[0] = o;
    /* evaluate the affine map even when not owned (barycentrics may be negative) */
    for (int k = 0; k < 4; k++) e[k] = face_eval(&F, k, q);
    int so = 1 - s;
    i128 M = (i128)1024 * F.absdet, Pnum[3];
    double xp[3];
    for (int a = 0; a < 3; a++) {
        i128 Nn = 0;
        for (int k = 0; k < 4; k++) Nn += e[k] * (i128)(Q[so][k][a] - Q[s][k][a]);
        Pnum[a] = (i128)q[a] * M + Nn;
        xp[a] = (double)q[a] + (double)Nn / ((double)F.absdet * 1024.0);
        out[1 + a] = xp[a];
        int64_t st[2] = {0, 0};
        int c = axis_set(Pnum[a], M, P->n[a], st);
        sets[3 * a + 0] = c;
        sets[3 * a + 1] = st[0];
        sets[3 * a + 2] = c == 2 ? st[1] : -1;
    }
    int inimg = q[0] >= 0 && q[0] < P->n[0] && q[1] >= 0 && q[1] < P->n[1] && q[2] >= 0 && q[2] < P->n[2];
    out[4] = inimg ? (double)P->I[s][vidx(P, q[0], q[1], q[2])] : NAN;
    out[5] = trilinear(P, P->I[so], xp);
    out[6] = fg_exact(P, P->I[so], Pnum, M);
    out[7] = inimg ? h_of(out[4], out[5], (int)out[6]) : NAN;
    return 0;
}

/* exported helpers for the pin tests (pure functions of their arguments) */
double orc_h(double a, double b, int fg) { return h_of(a, b, fg); }

/* NEXT-1 switches and pin hooks */
int orc_set_sampler(orc_problem *P, int mode, double rate) {
    if ((mode != 0 && mode != 1) || !(rate > 0.0)) return -1;
    P->sampler = mode;
    P->rate = rate;
    return 0;
}
void orc_sobol_point(uint64_t k, uint32_t *x4) {
    sobol_init();
    sobol_point(k, x4);
}
double orc_neg_log(uint32_t x) { return neg_log(x); }
double orc_det_ln(double r) { return det_ln(r); }
/* n standard normals in consecutive pairs from one key (P5 generator) */
void orc_gauss(uint64_t key, int n, double *out) {
    uint64_t ctr = 0;
    for (int i = 0; i + 1 < n + 1; i += 2) {
        double a, b;
        gauss_pair(key, &ctr, &a, &b);
        out[i] = a;
        if (i + 1 < n) out[i + 1] = b;
    }
}
double orc_repair_sigma(orc_problem *P, const float *off, int s, int j) { return repair_sigma(P, off, s, j); }
uint64_t orc_fnv1a64(const unsigned char *b, int64_t n) { return fnv1a64(b, (size_t)n); }
uint64_t orc_splitmix64(uint64_t z) { return splitmix64(z); }
/* M1/M2 sampler alone: x = mu + L z for (seed, gen, k, g), d variables (fp64) */
void orc_mix_sample(const double *mu, const double *L, int d, uint64_t seed, int64_t gen, int64_t k, int g,
                    double *x) {
    double *z = (double *)malloc(sizeof(double) * (d + 2));
    uint64_t key = mix_key(seed, gen, k, g), ctr = 0;
    for (int i = 0; i < d; i += 2) gauss_pair(key, &ctr, &z[i], &z[i + 1]);
    for (int i = 0; i < d; i++) {
        double v = mu[i];
        for (int j = 0; j <= i; j++) v = v + L[(int64_t)i * d + j] * z[j];
        x[i] = v;
    }
    free(z);
}
uint64_t orc_tet_seed(const int64_t *Q12, uint32_t *mask4) {
    int64_t Q[4][3];
    for (int k = 0; k < 4; k++)
        for (int a = 0; a < 3; a++) Q[k][a] = Q12[3 * k + a];
    tet_masks(Q, mask4);
    return tet_seed(Q);
}
/* sample k of tet t, side s: out = lambda[4], p[3], Tp[3], a, b, fa, fb, h, N */
int orc_sobol_debug(orc_problem *P, const float *offsets_one, int t, int s, int64_t k, double *out) {
    int64_t Q[2][4][3];
    if (t < 0 || t >= P->T || s < 0 || s > 1) return -1;
    if (!tet_coords(P, offsets_one, t, Q)) return -3;
    uint32_t x[4], mask[4];
    double lam[4], p[3], tp[3];
    tet_masks(Q[s], mask);
    sobol_point((uint64_t)k, x);
    sobol_lambda(x, mask, lam);
    bary_point(Q[s], lam, p);
    bary_point(Q[1 - s], lam, tp);
    double a = trilinear(P, P->I[s], p), b = trilinear(P, P->I[1 - s], tp);
    int fa = positive_at(P, P->I[s], p), fb = positive_at(P, P->I[1 - s], tp);
    for (int j = 0; j < 4; j++) out[j] = lam[j];
    for (int a2 = 0; a2 < 3; a2++) { out[4 + a2] = p[a2]; out[7 + a2] = tp[a2]; }
    out[10] = a; out[11] = b; out[12] = fa; out[13] = fb;
    out[14] = (fa && fb) ? (a - b) * (a - b) : ((!fa && !fb) ? 0.0 : 1.0);
    out[15] = (double)sobol_count(P, Q[s]);
    return 0;
}
double orc_trilinear_raw(int nx, int ny, int nz, const float *vol, double x, double y, double z) {
    orc_problem tmp;
    memset(&tmp, 0, sizeof(tmp));
    tmp.n[0] = nx; tmp.n[1] = ny; tmp.n[2] = nz;
    double p[3] = {x, y, z};
    return trilinear(&tmp, vol, p);
}
int orc_signed_det(const int64_t *Q12, int64_t *hi, uint64_t *lo) {
    int64_t Q[4][3];
    memcpy(Q, Q12, sizeof(Q));
    i128 d = det4(Q);
    *hi = (int64_t)(d >> 64);
    *lo = (uint64_t)d;
    return sgn128(d);
}
int64_t orc_canon(float b, float o) { return canon(b, o); }
int orc_ref_sign(const orc_problem *P, int t) { return P->ref[t]; }
double orc_r(const orc_problem *P) { return P->r; }

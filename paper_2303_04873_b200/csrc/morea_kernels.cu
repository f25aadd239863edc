// morea_kernels.cu -- sm_100a kernels of the MOREA hot path (arXiv 2303.04873).
//
// Rows of SURVEY.md §8(a) and where they live:
//   a0 load-time maps          k_distance_maps, k_band_mask, k_validate_volume
//   a1 genotype decode          canon_q (fp64, exact Q.10 rounding)
//   a2 per-tet geometry + fold  k_setup (build_side, folds, severity)
//   a3 magnitude                k_setup (magnitude)
//   a4 ownership rasterizer     k_raster: row_interval() + raster() (exact intervals)
//   a5 map + sample + h         k_raster: Sample<>::sample (exact case split, exact_fg)
//   a6 guidance term            k_raster: Sample<>::enqueue / entry (band bits, per-warp queue)
//   a7 reductions               warp shuffles (fixed order), k_reduce
//   a8 partial evaluation       version 0/1 items + k_reduce with base_acc
//   a9 fold check               k_check_folds
// The readings of the paper (O1..O13) are cited per function.
//
// Work decomposition.  k_setup: one thread per (version, tet,
// solution) computes the exact integer geometry of both sides (int64/int128)
// and writes a 384-byte SideRec per side.  k_raster: one 28-warp block per SM
// pulls chunks of up to 112 items from a global queue in solution-minor order
// and its warps take them one at a time without a block barrier (BlockQueue)
// (consecutive items = same tet, next solution, so the warps of an SM share
// their texel and record footprints in L1; large tets first).  Inside an item
// the 32 lanes compute the exact x-intervals of 32 bbox rows, prefix-sum their
// lengths and sweep the flattened samples 32 at a time.  The other volume is
// gathered with tld4 from edge-padded textures (the O5 clamp is needed only by
// items whose other-side vertices leave (-1, n), a separate instantiation).
// Hot paths carry no divergent branches: rare exact fallbacks sit behind
// warp-uniform votes, shared-memory records are written with predicated
// stores (DESIGN.md §4.4 lists what was measured and why).
// Further sm_100a kernels: morea_sobol*.cuh (NEXT-1 Sobol sampler),
// morea_repair.cuh (NEXT-2 fold repair), morea_mix.cuh (NEXT-3 optimal
// mixing), morea_export.cuh (NEXT-4 object counts and DVF).
#include <cuda_runtime.h>

#include <cstdint>

#include "morea.h"
#include "morea_internal.h"

#ifndef MOREA_SM_BLOCK
#define MOREA_SM_BLOCK 28  // k_raster: one block of this many warps per SM
#endif

#ifndef MOREA_SOBOL_WARPS
#define MOREA_SOBOL_WARPS 28  // k_sobol: warps of its one block per SM
#endif

#ifndef MOREA_CLAIM_CHUNK
#define MOREA_CLAIM_CHUNK 112  // k_raster, k_sobol: at most this many items per global claim of BlockQueue
#endif

#ifndef MOREA_CLAIM_SPREAD
#define MOREA_CLAIM_SPREAD 16  // k_raster, k_sobol: at least this many claims per block per launch where possible
#endif

namespace morea {

typedef long long i64;
typedef unsigned long long u64;
typedef __int128 i128;
#define FULLMASK 0xffffffffu

// ---------------------------------------------------------------------------
// a1: canonical coordinates (O1): Q = round-half-even(1024 B + 1024 O) in fp64.
// Both products are exact (power-of-two scaling of fp32 values); the sum is one
// IEEE rounding; __double2ll_rn rounds half to even.
// ---------------------------------------------------------------------------
__device__ __forceinline__ i64 canon_q(float b, float o) {
  double v = __dadd_rn(__dmul_rn(1024.0, (double)b), __dmul_rn(1024.0, (double)o));
  return __double2ll_rn(v);
}

__device__ __forceinline__ i64 det3(const int Q[4][3]) {
  i64 a0 = Q[1][0] - Q[0][0], a1 = Q[1][1] - Q[0][1], a2 = Q[1][2] - Q[0][2];
  i64 b0 = Q[2][0] - Q[0][0], b1 = Q[2][1] - Q[0][1], b2 = Q[2][2] - Q[0][2];
  i64 c0 = Q[3][0] - Q[0][0], c1 = Q[3][1] - Q[0][1], c2 = Q[3][2] - Q[0][2];
  return a0 * (b1 * c2 - b2 * c1) - a1 * (b0 * c2 - b2 * c0) + a2 * (b0 * c1 - b1 * c0);
}

__device__ __forceinline__ int floordiv1024(int v) { return v >> 10; }  // arithmetic shift = floor
__device__ __forceinline__ int ceildiv1024(int v) { return -((-v) >> 10); }

// Load + canonicalise the 4 vertices of a tet on both sides.  Returns false if
// a vertex is outside the Q.10 window (flag DOMAIN).
__device__ __forceinline__ bool load_tet(const EvalArgs& A, int sol, int4 tv, int4 slots,
                                         int Q[2][4][3]) {
  const int vid[4] = {tv.x, tv.y, tv.z, tv.w};
  const int sl[4] = {slots.x, slots.y, slots.z, slots.w};
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int j = vid[k];
    MOREA_CHECK(j >= 0 && j < A.mesh.N && sl[k] < A.S_total && sol >= 0 && sol < A.P);
    // the point's 6 offsets (24 contiguous bytes) as three 8-byte loads; the API
    // stages offsets / new values that are not 8-byte aligned
    const float2* o = reinterpret_cast<const float2*>(
        sl[k] >= 0 ? A.new_vals + ((long long)sol * A.S_total + sl[k]) * 6
                   : A.offsets + ((long long)sol * A.mesh.N + j) * 6);
    const float2 o01 = __ldg(o), o23 = __ldg(o + 1), o45 = __ldg(o + 2);
    const float oo[6] = {o01.x, o01.y, o23.x, o23.y, o45.x, o45.y};
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const float b = __ldg(&A.mesh.base[3 * j + a]);
#pragma unroll
      for (int s = 0; s < 2; s++) {
        const i64 q = canon_q(b, oo[3 * s + a]);
        ok = ok && (q >= kQLo) && (q < kQHi);
        Q[s][k][a] = (int)q;
      }
    }
  }
  return ok;
}

// ---------------------------------------------------------------------------
// a2: exact geometry of one side (O2, O3, O4).  |Q| < 2^19.6 so edge components
// < 2^20, normals < 2^41, |Delta| < 2^62.6, e_k(q) < 3 2^61.
// ---------------------------------------------------------------------------
__device__ void build_side_ordered(const int Q[4][3], const int Qo[4][3], int nx, int ny, int nz,
                                   SideRec& G) {
  G.flags = 0;
  const i64 det = det3(Q);
  if (det == 0) return;  // degenerate: owns nothing (O3)
  G.absdet = det < 0 ? -det : det;
  const int dims[3] = {nx, ny, nz};
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const int mn = min(min(Q[0][a], Q[1][a]), min(Q[2][a], Q[3][a]));
    const int mx = max(max(Q[0][a], Q[1][a]), max(Q[2][a], Q[3][a]));
    G.lo[a] = max(ceildiv1024(mn), 0);
    G.hi[a] = min(floordiv1024(mx), dims[a] - 1);
    if (G.lo[a] > G.hi[a]) return;  // no lattice point of the image inside
  }
  const double Ly = (double)(G.hi[1] - G.lo[1]), Lz = (double)(G.hi[2] - G.lo[2]);
#pragma unroll
  for (int k = 0; k < 4; k++) {
    G.vy[k] = (float)Q[k][1] * (1.0f / 1024.0f);  // exact: |Q| < 2^20
    G.vz[k] = (float)Q[k][2] * (1.0f / 1024.0f);
    const int f0 = (k == 0) ? 1 : 0;
    const int f1 = (k <= 1) ? 2 : 1;
    const int f2 = (k <= 2) ? 3 : 2;
    const i64 u0 = Q[f1][0] - Q[f0][0], u1 = Q[f1][1] - Q[f0][1], u2 = Q[f1][2] - Q[f0][2];
    const i64 v0 = Q[f2][0] - Q[f0][0], v1 = Q[f2][1] - Q[f0][1], v2 = Q[f2][2] - Q[f0][2];
    i64 n0 = u1 * v2 - u2 * v1, n1 = u2 * v0 - u0 * v2, n2 = u0 * v1 - u1 * v0;
    const i64 s = n0 * (Q[k][0] - Q[f0][0]) + n1 * (Q[k][1] - Q[f0][1]) + n2 * (Q[k][2] - Q[f0][2]);
    if (s < 0) { n0 = -n0; n1 = -n1; n2 = -n2; }  // inward: towards vertex k
    G.nrm[k][0] = n0; G.nrm[k][1] = n1; G.nrm[k][2] = n2;
    G.cst[k] = n0 * (i64)Q[f0][0] + n1 * (i64)Q[f0][1] + n2 * (i64)Q[f0][2];
#pragma unroll
    for (int a = 0; a < 3; a++) G.U[k][a] = Qo[k][a] - Q[k][a];
    // row crossing x*(y, z): 1024 (n0 x + n1 y + n2 z) = cst, evaluated in fp32 per row
    if (n0 != 0) {
      const i128 num = (i128)G.cst[k] - (i128)1024 * ((i128)n1 * G.lo[1] + (i128)n2 * G.lo[2]);
      // one fp64 reciprocal per face: the fp32 coefficients are within 2^-24 (1 + 2^-50)
      // of the exact ratios, inside the crossing bound thr below (4x the fp32 worst case)
      const double rn0 = 1.0 / (double)n0;
      const double fa = (double)num * rn0 * (1.0 / 1024.0);
      const double fb = -(double)n1 * rn0, fc = -(double)n2 * rn0;
      G.face[k].x = (float)fa;
      G.face[k].y = (float)fb;
      G.face[k].z = (float)fc;
      // fp32 rounding of 3 coefficients + 2 fma: < 2^-22 (|fa| + |fb| Ly + |fc| Lz); 4x margin
      const double thr = ldexp(fabs(fa) + fabs(fb) * Ly + fabs(fc) * Lz + 1.0, -20);
      G.face[k].w = (float)thr;
      G.ftype[k] = (n0 > 0 ? 1 : -1) * (thr >= 0.25 ? 2 : 1);
    } else {
      G.ftype[k] = 0;
      G.face[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  // O4: displacement u(p) = sum_k lambda_k(p) U_k / 1024, lambda_k = e_k / |Delta|.
  // Gradient du_a/dp_b = sum_k n_kb U_ka / |Delta|; value at lo from exact e_k(lo).
  const double inv_det = 1.0 / (double)G.absdet;
  const double L[3] = {(double)(G.hi[0] - G.lo[0]), Ly, Lz};
  i64 elo[4];
#pragma unroll
  for (int k = 0; k < 4; k++)
    elo[k] = 1024 * (G.nrm[k][0] * G.lo[0] + G.nrm[k][1] * G.lo[1] + G.nrm[k][2] * G.lo[2]) - G.cst[k];
  bool inside = true;   // positions in [0, n-1) (plain-load path needs no clamp)
  bool inside_p = true; // positions in (-1, n) (edge-padded textures need no clamp)
#pragma unroll
  for (int a = 0; a < 3; a++) {
    bool exact = true;
    double Aab[3];
#pragma unroll
    for (int b = 0; b < 3; b++) {
      // |n_kb| < 2^41, |U_ka| < 2^20 (Q.10 window): each product < 2^61, the sum of
      // four < 2^63, so int64 is exact
      i64 num = 0;
#pragma unroll
      for (int k = 0; k < 4; k++) num += G.nrm[k][b] * (i64)G.U[k][a];
      if (num != 0) exact = false;
      Aab[b] = (double)num * inv_det;
      G.A[a][b] = (float)Aab[b];
    }
    if (exact) {
      // every vertex moves by the same U_a: x_a = q_a + U_a / 1024 exactly (fp32-exact)
      G.d0[a] = (float)G.U[0][a] * (1.0f / 1024.0f);
      G.eps[a] = 0.0f;
    } else {
      i128 N = 0;
#pragma unroll
      for (int k = 0; k < 4; k++) N += (i128)elo[k] * (i128)G.U[k][a];
      const double d0 = (double)N / (1024.0 * (double)G.absdet);
      G.d0[a] = (float)d0;
      double amax = 0.0;
#pragma unroll
      for (int c = 0; c < 8; c++) {
        const double v = d0 + Aab[0] * ((c & 1) ? L[0] : 0.0) + Aab[1] * ((c & 2) ? L[1] : 0.0) +
                         Aab[2] * ((c & 4) ? L[2] : 0.0);
        amax = fmax(amax, fabs(v));
      }
      // fp32 error of d = fma(A_x0, k, d_row(fp32 fma chain)) and of frac(d):
      // <= 2^-24 (5 (|u|max + sum_b |A_ab| L_b) + 1); eps = 3x that
      const double bound = amax + fabs(Aab[0]) * L[0] + fabs(Aab[1]) * L[1] + fabs(Aab[2]) * L[2] + 1.0;
      G.eps[a] = (float)ldexp(bound, -19);
    }
    // An owned sample q lies in the closed tet, so its exact position x = T(q)
    // (a convex combination of the other side's vertices) lies in the other
    // side's vertex bbox.  The margin covers the fp32 position error, so floor()
    // of the fp32 position stays in range.
    const int omn = min(min(Qo[0][a], Qo[1][a]), min(Qo[2][a], Qo[3][a]));
    const int omx = max(max(Qo[0][a], Qo[1][a]), max(Qo[2][a], Qo[3][a]));
    const double xmin = (double)omn / 1024.0, xmax = (double)omx / 1024.0;
    const double mg = 1e-3 + 2.0 * (double)G.eps[a];
    if (!(xmin >= mg && xmax <= (double)(dims[a] - 1) - mg)) inside = false;
    if (!(xmin >= -1.0 + mg && xmax <= (double)dims[a] - mg)) inside_p = false;
  }
  bool regular = true;
#pragma unroll
  for (int k = 0; k < 4; k++) regular = regular && (G.ftype[k] == 1 || G.ftype[k] == -1);
  // Regular items list their lower-bound faces (n_x > 0) first (build_side orders the
  // vertices so), nl of them.  The fast row interval (row_interval) takes the max of
  // the crossings of faces [0, nl) and the min of faces [nl, 4) with no per-face
  // selects; its ambiguity test needs the binding crossing's bound, so each group's
  // bounds widen to the group maximum.
  int nl = 0;
  if (regular) {
    while (nl < 4 && G.ftype[nl] > 0) nl++;
    regular = nl >= 1 && nl <= 3;
#pragma unroll
    for (int k = 1; k < 4; k++) regular = regular && (G.ftype[k] <= G.ftype[k - 1]);
  }
  if (regular) {
    float wl = 0.f, wh = 0.f;
#pragma unroll
    for (int k = 0; k < 4; k++) {
      if (k < nl) wl = fmaxf(wl, G.face[k].w);
      else wh = fmaxf(wh, G.face[k].w);
    }
#pragma unroll
    for (int k = 0; k < 4; k++) G.face[k].w = k < nl ? wl : wh;
  } else {
    nl = 0;
  }
  // Empty-space radius (bits 8..15): an owned sample q maps to x = q + u(q) with u a
  // convex combination of the vertex displacements, so |u_a| <= max_k |U_ka| / 1024 and
  // every trilinear corner of x lies within Chebyshev distance R - 1 of q, R =
  // ceil(max |U| / 1024) + 2.  If the other volume is zero on that box and I(q) = 0,
  // h = 0 exactly (no contributing corner is > 0), whatever the position's rounding.
  int maxU = 0;
#pragma unroll
  for (int k = 0; k < 4; k++)
#pragma unroll
    for (int a = 0; a < 3; a++) maxU = max(maxU, abs(G.U[k][a]));
  const int skipR = min((maxU + 1023) / 1024 + 2, 255);
  G.flags = 1 | (inside ? 2 : 0) | (regular ? 4 : 0) | (inside_p ? 8 : 0) | (skipR << 8) | (nl << 16);
}

// Orders the vertices so that the faces opposite them that bound x from below (inward
// n_x > 0) come first, then the rest (a stable partition of a local copy; face k stays
// opposite vertex k, so U_k and e_k keep their pairing), and builds the side record.
// Vertex order changes nothing else the record holds.
__device__ void build_side(const int Q[4][3], const int Qo[4][3], int nx, int ny, int nz, SideRec& G) {
  int low = 0;  // bit k: the face opposite vertex k is a lower bound along x
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int f0 = (k == 0) ? 1 : 0;
    const int f1 = (k <= 1) ? 2 : 1;
    const int f2 = (k <= 2) ? 3 : 2;
    const i64 u0 = Q[f1][0] - Q[f0][0], u1 = Q[f1][1] - Q[f0][1], u2 = Q[f1][2] - Q[f0][2];
    const i64 v0 = Q[f2][0] - Q[f0][0], v1 = Q[f2][1] - Q[f0][1], v2 = Q[f2][2] - Q[f0][2];
    const i64 n0 = u1 * v2 - u2 * v1, n1 = u2 * v0 - u0 * v2, n2 = u0 * v1 - u1 * v0;
    const i64 sd = n0 * (Q[k][0] - Q[f0][0]) + n1 * (Q[k][1] - Q[f0][1]) + n2 * (Q[k][2] - Q[f0][2]);
    if ((sd < 0 ? -n0 : n0) > 0) low |= 1 << k;
  }
  int src[4], c = 0;
#pragma unroll
  for (int k = 0; k < 4; k++)
    if (low >> k & 1) src[c++] = k;
#pragma unroll
  for (int k = 0; k < 4; k++)
    if (!(low >> k & 1)) src[c++] = k;
  int P[4][3], Po[4][3];
#pragma unroll
  for (int k = 0; k < 4; k++)
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const int j = src[k];
      P[k][a] = j == 0 ? Q[0][a] : j == 1 ? Q[1][a] : j == 2 ? Q[2][a] : Q[3][a];
      Po[k][a] = j == 0 ? Qo[0][a] : j == 1 ? Qo[1][a] : j == 2 ? Qo[2][a] : Qo[3][a];
    }
  build_side_ordered(P, Po, nx, ny, nz, G);
}

// ---------------------------------------------------------------------------
// a3: magnitude (O9), fp64 from exact integer edge vectors.
// (L_s - L_t) = (S_s - S_t) / (sqrt S_s + sqrt S_t), S = sum_a s_a^2 D_a^2.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double edge_term(const i64 ds[3], const i64 dt[3], const double sp2[3],
                                            double scale) {
  double Ss = 0.0, St = 0.0, diff = 0.0;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    Ss += sp2[a] * (double)(ds[a] * ds[a]);
    St += sp2[a] * (double)(dt[a] * dt[a]);
    diff += sp2[a] * (double)(ds[a] * ds[a] - dt[a] * dt[a]);
  }
  const double den = sqrt(Ss) + sqrt(St);
  const double d = den > 0.0 ? diff / den * scale : 0.0;
  return d * d;
}

__device__ double magnitude(const int Q[2][4][3], double c, const double sp2[3], int spoke_mode) {
  double m = 0.0;
  const int E[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
#pragma unroll
  for (int e = 0; e < 6; e++) {
    i64 ds[3], dt[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      ds[a] = (i64)Q[0][E[e][0]][a] - Q[0][E[e][1]][a];
      dt[a] = (i64)Q[1][E[e][0]][a] - Q[1][E[e][1]][a];
    }
    m += edge_term(ds, dt, sp2, 1.0 / 1024.0);
  }
  // spokes: vertex -> centroid of the opposite face = (3 v - sum of the others) / 3
  const double ss = (spoke_mode == 1 ? 0.75 : 1.0) / 3072.0;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    i64 ds[3], dt[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      ds[a] = 4 * (i64)Q[0][k][a] - ((i64)Q[0][0][a] + Q[0][1][a] + Q[0][2][a] + Q[0][3][a]);
      dt[a] = 4 * (i64)Q[1][k][a] - ((i64)Q[1][0][a] + Q[1][1][a] + Q[1][2][a] + Q[1][3][a]);
    }
    m += edge_term(ds, dt, sp2, ss);
  }
  return c * m;
}

#include "morea_sobol_setup.cuh"

// ---------------------------------------------------------------------------
// k_setup: one thread per (version, canonical entry, solution).  The SideRecs are
// built in a per-warp shared-memory stage (a 400-byte slot per lane: bank-conflict
// free 16-byte stores) and copied out by the whole warp, side by side: the 32
// records of one side of a warp's items land as 384-byte runs (coalesced) instead of
// one thread storing 24 scattered 16-byte words.
// ---------------------------------------------------------------------------
constexpr int kSetupThreads = 128;
constexpr int kStageVec = (int)(sizeof(SideRec) / 16) + 1;  // 25 int4 per lane slot
constexpr size_t kSetupSmem = (size_t)kSetupThreads * kStageVec * 16;

__global__ void __launch_bounds__(kSetupThreads, 3) k_setup(const EvalArgs A) {
  extern __shared__ int4 setup_stage[];
  const int lane = threadIdx.x & 31;
  int4* stage = setup_stage + (threadIdx.x >> 5) * 32 * kStageVec;
  SideRec& G = *reinterpret_cast<SideRec*>(stage + lane * kStageVec);
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per_v = (long long)A.n_entries * A.P;
  int Q[2][4][3];
  int mode = 0;  // SideRec path: 1 = build both sides, 2 = domain error (flags 0), 0 = none
  if (i < per_v * A.n_setup_versions) {
    const int v = (int)(i / per_v);
    const long long rem = i - (long long)v * per_v;
    const int e = (int)(rem / A.P);
    const int sol = (int)(rem - (long long)e * A.P);
    const int tet = A.canon_tet ? A.canon_tet[e] : e;
    const int4 none = make_int4(-1, -1, -1, -1);
    const int4 slots = (v == 0 && A.canon_slots) ? A.canon_slots[e] : none;
    Scal sc;
    sc.m = sc.sev = 0.0;
    sc.folds = sc.flags = 0;
    sc.pad[0] = sc.pad[1] = 0;
    const bool raster = v < A.n_raster_versions;
    if (!load_tet(A, sol, A.mesh.tets[tet], slots, Q)) {
      sc.flags = 1;  // domain: the tet contributes nothing
      A.scal[i] = sc;
      if (raster) {
        if (A.sampler == 1) {
          A.sgeom[2 * i].flags = 0;
          A.sgeom[2 * i + 1].flags = 0;
        } else {
          mode = 2;
        }
      }
    } else {
      const Volumes& V = A.vol;
      const double sp2[3] = {V.sp[0] * V.sp[0], V.sp[1] * V.sp[1], V.sp[2] * V.sp[2]};
      sc.m = magnitude(Q, (double)A.mesh.cdelta[tet], sp2, A.mesh.spoke_mode);
      const int ref = A.mesh.ref[tet];
#pragma unroll
      for (int s = 0; s < 2; s++) {
        const i64 det = det3(Q[s]);
        const int sg = (det > 0) - (det < 0);
        if (sg != ref) {  // O2: sign change w.r.t. the reference sign; zero counts as a fold
          sc.folds += 1;
          const double vol = (double)(det < 0 ? -det : det) / (6.0 * 1073741824.0);
          sc.sev += vol * V.sp[0] * V.sp[1] * V.sp[2];
        }
      }
      if (raster && A.sampler == 1) {
#pragma unroll 1
        for (int s = 0; s < 2; s++) {
          SobolRec SG;
          build_sobol(Q[s], Q[1 - s], V, A.rate, SG);
          if (SG.N > 0x7fffffffLL) {  // beyond the 32-bit point counter: flagged like a domain
            sc.flags = 1;             // error (objectives NaN), the side contributes nothing
            SG.flags = 0;
          }
          const int4* src = reinterpret_cast<const int4*>(&SG);
          int4* dst = reinterpret_cast<int4*>(&A.sgeom[2 * i + s]);
#pragma unroll
          for (int t = 0; t < (int)(sizeof(SobolRec) / 16); t++) dst[t] = src[t];
        }
      } else if (raster) {
        mode = 1;
      }
      A.scal[i] = sc;
    }
  }
  if (A.sampler == 1) return;  // kernel-uniform
  const unsigned wm = __ballot_sync(FULLMASK, mode != 0);
  if (!wm) return;  // warp-uniform
  const long long i0 = i - lane;  // the warp's first item
#pragma unroll 1
  for (int s = 0; s < 2; s++) {
    if (mode == 1) build_side(Q[s], Q[1 - s], A.vol.nx, A.vol.ny, A.vol.nz, G);
    else if (mode == 2) G.flags = 0;
    __syncwarp();
    // record j of the stage -> A.geom[2 (i0 + j) + s], 24 int4 each, 32 lanes at a time:
    // word m = 24 j + t sits at stage[m + j] and at byte 16 m + 384 j from side s's
    // first record (records of one side are 768 bytes apart)
    char* const dst0 = reinterpret_cast<char*>(&A.geom[2 * i0 + s]);
#pragma unroll 4
    for (int m = lane; m < 32 * (kStageVec - 1); m += 32) {
      const int j = m / (kStageVec - 1);
      if (wm >> j & 1u) *reinterpret_cast<int4*>(dst0 + (16 * m + 384 * j)) = stage[m + j];
    }
    __syncwarp();
  }
}

// the 50 KB stage needs the opt-in above 48 KB (morea_create, per context's device)
cudaError_t setup_prepare() {
  return cudaFuncSetAttribute(k_setup, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSetupSmem);
}

cudaError_t launch_setup(const EvalArgs& a, cudaStream_t s) {
  const long long n = (long long)a.n_setup_versions * a.n_entries * a.P;
  if (n == 0) return cudaSuccess;
  k_setup<<<(unsigned)((n + kSetupThreads - 1) / kSetupThreads), kSetupThreads, kSetupSmem, s>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// a4: exact x-interval of owned lattice points on row (y, z) (O3).  Face k owns
// q iff e_k(q) > 0, or e_k = 0 and lexpos(n_k) (perturbation q + (e, e^2, e^3)).
// Along x, e_k(x) = 1024 n_kx x + const: a half-line bounded at the crossing
// x*, evaluated in fp64; exact int64 evaluation only when x* is within the
// (tiny) fp64 error bound of an integer.
// ---------------------------------------------------------------------------
__device__ __forceinline__ i64 face_e(const SideRec& R, int k, int x, int y, int z) {
  return 1024 * (R.nrm[k][0] * x + R.nrm[k][1] * y + R.nrm[k][2] * z) - R.cst[k];
}

__device__ __noinline__ void row_interval_exact(const SideRec& R, int y, int z, int& xl, int& xh) {
  const int lo = R.lo[0], hi = R.hi[0];
  xl = lo;
  xh = hi;
  const float dy = (float)(y - R.lo[1]), dz = (float)(z - R.lo[2]);
  const int4 types = *reinterpret_cast<const int4*>(R.ftype);
  const int tk[4] = {types.x, types.y, types.z, types.w};
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int t = tk[k];
    if (t == 0) {
      const i64 E = face_e(R, k, 0, y, z);
      const bool own = E > 0 || (E == 0 && (R.nrm[k][1] > 0 || (R.nrm[k][1] == 0 && R.nrm[k][2] > 0)));
      if (!own) xh = lo - 1;
      continue;
    }
    const float4 fc4 = R.face[k];
    float xs = fmaf(fc4.z, dz, fmaf(fc4.y, dy, fc4.x));
    xs = fminf(fmaxf(xs, (float)lo - 4.5f), (float)hi + 4.5f);
    const float xr = rintf(xs);
    if (t == 2 || t == -2) {  // exact monotone search (rare: nearly x-parallel face)
      int x = (int)xr;
      if (t > 0) {  // smallest x in [lo, hi+1] with e >= 0
        x = min(max(x, lo), hi + 1);
        while (x > lo && face_e(R, k, x - 1, y, z) >= 0) --x;
        while (x <= hi && face_e(R, k, x, y, z) < 0) ++x;
        xl = max(xl, x);
      } else {      // largest x in [lo-1, hi] with e > 0
        x = min(max(x, lo - 1), hi);
        while (x < hi && face_e(R, k, x + 1, y, z) > 0) ++x;
        while (x >= lo && face_e(R, k, x, y, z) <= 0) --x;
        xh = min(xh, x);
      }
      continue;
    }
    int xi;
    if (fabsf(xs - xr) > fc4.w) {
      xi = (int)ceilf(xs) - (t < 0 ? 1 : 0);  // lower: smallest x > x*; upper: largest x < x*
    } else {  // x* within the error bound of the integer c: decide exactly
      const int c = (int)xr;
      const i64 e = face_e(R, k, c, y, z);
      xi = t > 0 ? (e >= 0 ? c : c + 1) : (e > 0 ? c : c - 1);
    }
    if (t > 0) xl = max(xl, xi);
    else xh = min(xh, xi);
  }
}

// all lanes call it (warp-uniform branch); lanes with ex = false keep (xl, xh)
__device__ __noinline__ int2 row_interval_exact_if(bool ex, const SideRec& R, int y, int z, int xl, int xh) {
  if (ex) row_interval_exact(R, y, z, xl, xh);
  return make_int2(xl, xh);
}

// Fast path for items whose four faces are regular (n_x != 0, small crossing
// error bound): four fp32 crossings; the exact routine only when a crossing is
// within its bound of an integer.  Warp-collective: every lane calls it (rv:
// the lane's row is real), the exact routine runs under a warp-uniform branch.
__device__ __forceinline__ void row_interval(const SideRec& R, int y, int z, bool rv, int& xl, int& xh) {
  if (__all_sync(FULLMASK, !(R.flags & 4))) {  // item-uniform (R in shared memory)
    const int2 r = row_interval_exact_if(rv, R, y, z, R.lo[0], R.hi[0]);
    xl = r.x;
    xh = r.y;
    return;
  }
  const int lo = R.lo[0], hi = R.hi[0];
  const float dy = (float)(y - R.lo[1]), dz = (float)(z - R.lo[2]);
  // faces [0, nl) bound x from below, [nl, 4) from above (k_setup order, 1 <= nl <= 3):
  // owned x > max of the lower crossings and x < min of the upper ones.  Only the
  // binding crossing's rounding matters, so the ambiguity test is on the max / min
  // against the group's error bound (faces 0 and 3 carry them).
  const int nl = (R.flags >> 16) & 3;
  const float4 f0 = R.face[0], f1 = R.face[1], f2 = R.face[2], f3 = R.face[3];
  const float x0 = fmaf(f0.z, dz, fmaf(f0.y, dy, f0.x)), x1 = fmaf(f1.z, dz, fmaf(f1.y, dy, f1.x));
  const float x2 = fmaf(f2.z, dz, fmaf(f2.y, dy, f2.x)), x3 = fmaf(f3.z, dz, fmaf(f3.y, dy, f3.x));
  float ml = fmaxf(x0, fmaxf(nl > 1 ? x1 : x0, nl > 2 ? x2 : x0));
  float mh = fminf(x3, fminf(nl < 3 ? x2 : x3, nl < 2 ? x1 : x3));
  // no clamp to the bbox: the fp32 error bound (thr) holds for every row of the
  // item, |x*| < 2^19 for regular faces (thr < 1/4), and the max / min with lo, hi
  // below bound the interval; a crossing far outside the bbox that happens to lie
  // near an integer only sends the row to the exact routine
  bool amb = (fabsf(ml - rintf(ml)) <= f0.w) || (fabsf(mh - rintf(mh)) <= f3.w);
  // lower: smallest x > x*; upper: largest x < x* = ceil(x*) - 1
  xl = max(lo, __float2int_ru(ml));
  xh = min(hi, __float2int_ru(mh) - 1);
  amb = amb && rv;
  if (__any_sync(FULLMASK, amb)) {
    const int2 r = row_interval_exact_if(amb, R, y, z, xl, xh);
    xl = r.x;
    xh = r.y;
  }
}

// Conservative y range of the tet's cross-section with the plane z, from the
// item's edge table (WarpSmem::edge, built by load_rec: per edge its z range, the
// y at its lower end and dy/dz).  The exact vertex coordinates are fp32-exact, so
// an edge point y = y_lo + (z - z_lo) s errs by |y - y_lo| 2^-24 (the rounded
// slope) plus one rounding, < 2e-4 voxels: inside the 1e-3 voxel margin.
template <class WS>
__device__ __forceinline__ int2 slice_y_range(const WS& S, int z) {
  float ymin = 3.0e38f, ymax = -3.0e38f;
  const float zf = (float)z;
#pragma unroll
  for (int e = 0; e < 6; e++) {
    const float4 a = S.edge[e];  // (z_lo, z_hi, y at z_lo, dy/dz; 0 for a horizontal edge)
    const float b = S.edge_y1[e];  // horizontal edge: the other end's y; else NaN
    const bool in = zf >= a.x && zf <= a.y;
    const float y = fmaf(zf - a.x, a.w, a.z);
    // fminf / fmaxf return the non-NaN operand
    ymin = in ? fminf(ymin, fminf(y, b)) : ymin;
    ymax = in ? fmaxf(ymax, fmaxf(y, b)) : ymax;
  }
  return make_int2(max(S.R.lo[1], (int)ceilf(fmaxf(ymin - 1e-3f, -1.0e6f))),
                   min(S.R.hi[1], (int)floorf(fminf(ymax + 1e-3f, 1.0e6f))));
}

constexpr int kQueueCap = 64;     // < 32 pending + one round of <= 32
// per-warp shared memory <= 3.5 KB, so the 28-warp block stays <= 99 KB (the
// 100 KB carve-out step; see kRasterDynSmem)
constexpr int kStartWords = 32;  // row-start bitmap window: 1024 samples

struct WarpSmem {
  SideRec R;
  unsigned starts[kStartWords];  // row-start bitmap of the current row chunk
  float4 edge[6];    // the item side's edges for slice y ranges (load_rec, slice_y_range)
  float edge_y1[6];
  int4 row_a[32];    // (exclusive prefix, linear index of row start, dx0, dy0 as float bits)
  float4 row_b[32];  // (dz0, xl, y, z): fp32 displacement z at the row start, row start as floats
  float4 sc0, sc1;   // per-side sample constants (see Sample)
  int2 slices[32];   // non-empty z-slices of the current 32-slice chunk: (first row, ylo | slice << 16)
  unsigned long long stat[4];  // samples, band entries, items, skipped samples of this warp (profiling)
  unsigned swept;  // samples swept in the current item (profiling; lane 0)
  // band-entry queue of the guidance term (a6): entries are evaluated 32 at a time
  float4 qa[kQueueCap];  // (u, v, fx, fy): footprint texel coordinates and weights
  int2 qb[kQueueCap];    // (fz bits, own linear index)
  unsigned char qi[kQueueCap];  // pair i
};

// inclusive warp prefix sum; the shuffle's own in-range predicate guards the add
// (no per-step lane compare and select)
__device__ __forceinline__ int warp_incl_scan(int v, int) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
    asm("{\n .reg .s32 t;\n .reg .pred p;\n shfl.sync.up.b32 t|p, %0, %1, 0, -1;\n @p add.s32 %0, %0, t;\n}"
        : "+r"(v)
        : "r"(o));
  return v;
}


// Generic rasterizer: visits every owned sample of the side.  Rows are
// enumerated per z-slice over the slice's y range, 32 rows per step (lanes
// compute the exact x-intervals); non-empty rows are compacted into shared
// memory and their flattened samples are swept 32 per step.  A lane finds its
// row from the shared-memory bitmap of row starts: one broadcast word per
// 32-sample window and a popc.  Lanes past the end evaluate sample 0 of the last row with
// valid = false (no divergence).  All lanes of the warp must call it.
template <class F>
__device__ __forceinline__ void raster(const SideRec& R, int nx, int ny, int loff, WarpSmem& S,
                                       int lane, F& f) {
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int z0 = R.lo[2]; z0 <= R.hi[2]; z0 += 32) {
    const int zl = z0 + lane;
    const int2 yr = slice_y_range(S, zl);  // every lane; masked below
    const int ylo = yr.x, yhi = yr.y;
    const int cnt = zl <= R.hi[2] ? max(0, yhi - ylo + 1) : 0;
    const int zincl = warp_incl_scan(cnt, lane);
    const int nrows = __shfl_sync(FULLMASK, zincl, 31);
    // non-empty slices of the chunk, compacted: (first row, ylo, slice) by rank
    const int zstart = zincl - cnt;
    const bool zne = cnt > 0;
    {
      const unsigned nem = __ballot_sync(FULLMASK, zne);
      const unsigned addr = (unsigned)__cvta_generic_to_shared(&S.slices[__popc(nem & lt_mask)]);
      __syncwarp();
      // ylo < 768 (Q.10 window) and the slice index < 32 share one word
      asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %0, 0;\n @p st.shared.v2.b32 [%1], {%2, %3};\n}"
                   :
                   : "r"((unsigned)zne), "r"(addr), "r"(zstart), "r"(ylo | (lane << 16))
                   : "memory");
      __syncwarp();
    }
    // the lane's slice start for the row lookup; empty slices never match (one
    // value across the row loop instead of two)
    const int zs = zne ? zstart : 0x7fffffff;
    const unsigned le_mask0 = (2u << lane) - 1u;
    for (int r0 = 0; r0 < nrows; r0 += 32) {
      const int r = r0 + lane;
      // the lane's slice: rank = (non-empty slices starting before r0) + (slice
      // starts in [r0, r]) - 1, from one OR-reduction of start bits and a ballot
      const unsigned sb =
          __reduce_or_sync(FULLMASK, (zs >= r0 && zs < r0 + 32) ? (1u << (zs - r0)) : 0u);
      const int before = __popc(__ballot_sync(FULLMASK, zs < r0));
      MOREA_CHECK(before + __popc(sb & le_mask0) - 1 >= 0 && before + __popc(sb & le_mask0) - 1 < 32);
      const int2 sl = S.slices[before + __popc(sb & le_mask0) - 1];
      int xl, xh;
      const int z = z0 + (sl.y >> 16);
      const int y = (sl.y & 0xffff) + (r - sl.x);
      const bool rv = r < nrows;
      // the row's hull (quiet rows, below) is loaded before the interval is
      // computed, so its latency overlaps the interval arithmetic
      const int qo = F::kQuiet ? f.quiet_off() : -1;  // item-uniform; -1: radius beyond the hulls
      unsigned hbw = 0xffff0000u;  // packed hull (first | last << 16); (0, -1): empty
      if (F::kQuiet && qo >= 0)  // unconditional load (lanes past the chunk read the plane's first row)
        hbw = f.quiet_hull(qo + (rv ? z * ny + y : 0));
      row_interval(R, y, z, rv, xl, xh);  // every lane (warp-collective)
      const int len_all = rv ? max(0, xh - xl + 1) : 0;
      // quiet rows (empty space): every voxel of the row is background
      // with no band entry and the other volume is zero within the item's radius, so
      // each sample's h is exactly 0 -- counted, not swept.  The row is quiet when
      // [xl, xh] lies outside the hull of the image row's non-quiet voxels.
      int len = len_all;
      // the hull's halves are sign-extended by PRMTs that also read xh / xl, so they
      // are scheduled after the interval and the hull load's latency stays hidden
      int hx, hy;
      asm("prmt.b32 %0, %1, %2, 0x9910;" : "=r"(hx) : "r"(hbw), "r"(xh));
      asm("prmt.b32 %0, %1, %2, 0xBB32;" : "=r"(hy) : "r"(hbw), "r"(xl));
      if (F::kQuiet && qo >= 0 && len_all > 0 && (xh < hx || xl > hy)) {
        len = 0;
        f.quiet_row((z * ny + y) * nx + xl, len_all);  // 2 V < 2^31 (own-record index is an int)
      }
      // every sample counts (n), per lane: the item's warp reduction sums the lanes.
      // Quiet samples (profiling) = the item's samples - the swept ones (count_quiet
      // adds the swept ones, k_raster takes the difference per item)
      f.count_only(len_all);
      const unsigned ne = __ballot_sync(FULLMASK, len > 0);
      if (ne == 0u) continue;  // nothing to sweep: no prefix sum
      const int incl = warp_incl_scan(len, lane);
      const int total = __shfl_sync(FULLMASK, incl, 31);
      if (F::kQuiet && lane == 0) f.count_quiet(total);
      const int start = incl - len;
      __syncwarp();
      {
        // every lane computes its row record; lanes with a non-empty row store it
        // (predicated stores: no divergent branch)
        const int c = __popc(ne & lt_mask);
        const float ox = (float)(xl - R.lo[0]), oy = (float)(y - R.lo[1]), oz = (float)(z - R.lo[2]);
        float4 drow;
        drow.x = fmaf(R.A[0][2], oz, fmaf(R.A[0][1], oy, fmaf(R.A[0][0], ox, R.d0[0])));
        drow.y = fmaf(R.A[1][2], oz, fmaf(R.A[1][1], oy, fmaf(R.A[1][0], ox, R.d0[1])));
        drow.z = fmaf(R.A[2][2], oz, fmaf(R.A[2][1], oy, fmaf(R.A[2][0], ox, R.d0[2])));
        const unsigned ra_addr = (unsigned)__cvta_generic_to_shared(&S.row_a[c]);
        const unsigned rb_addr = (unsigned)__cvta_generic_to_shared(&S.row_b[c]);
        asm volatile(
            "{\n .reg .pred p;\n setp.gt.s32 p, %0, 0;\n"
            " @p st.shared.v4.b32 [%1], {%3, %4, %5, %6};\n"
            " @p st.shared.v4.f32 [%2], {%7, %8, %9, %10};\n}"
            :
            : "r"(len), "r"(ra_addr), "r"(rb_addr), "r"(start), "r"((z * ny + y) * nx + xl + loff),
              "r"(__float_as_int(drow.x)), "r"(__float_as_int(drow.y)), "f"(drow.z), "f"((float)xl),
              "f"((float)y), "f"((float)z)
            : "memory");
      }
      // Sweep in windows of 32 kStartWords samples.  The bitmap holds the row
      // starts of the window (bit s of word s/32); a lane's row is the number of
      // starts <= its sample index, minus one.  Past the end that is the last row
      // (no starts there), evaluated with valid = false.  The fp32 partial sums
      // are flushed once 16 or more steps accumulated (steps_done), across chunks.
      int rprev = -1;
      for (int base = 0; base < total; base += 32 * kStartWords) {
        const int nw = min(kStartWords, (total - base + 31) >> 5);
        __syncwarp();
        // clear the whole bitmap window: one 16-byte store per lane
        static_assert(kStartWords == 32, "one word per lane clears the window");
        S.starts[lane] = 0u;
        __syncwarp();
        if (len > 0 && start >= base && start < base + 32 * kStartWords)
          atomicOr(&S.starts[(start - base) >> 5], 1u << (start & 31));
        __syncwarp();
        for (int w = 0; w < nw; w++) {
          MOREA_CHECK(w >= 0 && w < kStartWords);
          const unsigned M = S.starts[w];
          unsigned lem;  // lanes <= this one (special register: no recomputation)
          asm("mov.u32 %0, %%lanemask_le;" : "=r"(lem));
          const int row = rprev + __popc(M & lem);
          rprev += __popc(M);
          const int idx = base + (w << 5) + lane;
          const bool valid = idx < total;
          MOREA_CHECK(row >= 0 && row < 32);
          const int4 ra = S.row_a[row];
          f.sample(ra, S.row_b[row], valid ? idx - ra.x : 0, valid);
        }
        f.steps_done(nw);
      }
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// O6 slow path: exact contributing corner set when the fp32 position is within
// eps of a lattice plane on some axis.  x_a = (q_a M + N_a) / M exactly, with
// M = 1024 |Delta| and N_a = sum_k e_k(q) U_ka (int128).
// ---------------------------------------------------------------------------
__device__ __noinline__ bool exact_fg(const SideRec& R, int qx, int qy, int qz, float dx, float dy,
                                      float dz, const float* __restrict__ vol, int nx, int ny,
                                      int nz) {
  const int q[3] = {qx, qy, qz};
  const float d[3] = {dx, dy, dz};
  const int dims[3] = {nx, ny, nz};
  i64 e[4];
  for (int k = 0; k < 4; k++) e[k] = face_e(R, k, qx, qy, qz);
  const i128 M = (i128)1024 * (i128)R.absdet;
  int cnt[3], idx[3][2];
  for (int a = 0; a < 3; a++) {
    i128 N = 0;
    for (int k = 0; k < 4; k++) N += (i128)e[k] * (i128)R.U[k][a];
    const i128 Pn = (i128)q[a] * M + N;
    if (Pn <= 0) {
      cnt[a] = 1; idx[a][0] = 0;
    } else if (Pn >= (i128)(dims[a] - 1) * M) {
      cnt[a] = 1; idx[a][0] = dims[a] - 1;
    } else {
      i64 k0 = (i64)q[a] + (i64)floorf(d[a]);
      while (Pn < (i128)k0 * M) --k0;
      while (Pn >= (i128)(k0 + 1) * M) ++k0;
      idx[a][0] = (int)k0;
      if (Pn == (i128)k0 * M) {
        cnt[a] = 1;
      } else {
        cnt[a] = 2; idx[a][1] = (int)k0 + 1;
      }
    }
  }
  for (int k = 0; k < cnt[2]; k++)
    for (int j = 0; j < cnt[1]; j++)
      for (int i = 0; i < cnt[0]; i++)
        if (__ldg(&vol[((long long)idx[2][k] * ny + idx[1][j]) * nx + idx[0][i]]) > 0.0f) return true;
  return false;
}

// all lanes of the warp call it (warp-uniform branch); lanes without an
// ambiguous position keep their fg
__device__ __noinline__ bool exact_fg_if(bool amb, bool fg, const SideRec& R, int qx, int qy, int qz,
                                         float dx, float dy, float dz, const float* __restrict__ vol,
                                         int nx, int ny, int nz) {
  if (!amb) return fg;
  return exact_fg(R, qx, qy, qz, dx, dy, dz, vol, nx, ny, nz);
}

__device__ __forceinline__ float lerpf(float a, float b, float t) { return fmaf(t, b - a, a); }

// Positivity-exact lerp: (1 - t) a + t b as fma(t, b, (1 - t) a).  For a, b >= 0
// and t in [0, 1] it is > 0 iff a contributing value (a with t < 1, b with
// t > 0) is > 0, barring underflow (excluded by the value precondition of
// morea_load_images: non-zero intensities >= 2^-40).
__device__ __forceinline__ float plerp(float a, float b, float t, float omt) {
  return fmaf(t, b, omt * a);
}

// a5 + a6: one sample of side SIDE.  The footprint weights are exact: 0 / 1 on
// clamped axes and exact-integer axes, and in [eps, 1 - eps] otherwise unless the
// position is ambiguous (then exact_fg decides), so fg = (b > 0) is exact.
// Volume pointers and texture handles are read from the kernel parameters with
// compile-time offsets (constant bank): no registers, and texture handles are
// provably warp-uniform (no waterfall loop around tld4).
struct Acc {
  // per-lane fp64 sums of h and of the guidance term, kept in local memory (touched
  // once per flush): two fewer registers in the sweep, whose register pressure
  // otherwise spills the row-chunk state (1.2% measured)
  volatile double* hg;
  float hf;     // fp32 partial sum of h over at most 47 steps (flushed into h)
  float gf;     // fp32 partial sum of guidance terms since the last flush (into g)
  int n;        // samples
  int qn;       // band entries in the per-warp queue (warp-uniform)
  int ns;       // sweep steps since the last flush (warp-uniform)
};

template <bool TEX, int SIDE_T, bool CLAMP, bool DUMP>
struct Sample {
  const Volumes& V;
  const SideRec& R;
  WarpSmem& S;
  const float4& sc0;  // shared: (A_x0, A_y0, A_z0, 0.5 - eps_x)  displacement gradient along x
  const float4& sc1;  // shared: (0.5 - eps_y, 0.5 - eps_z, uoff, -): ambiguity thresholds on
                      // |f - 0.5|; uoff = texel x offset of corner i0 + 1 in the gather layout
  Acc& acc;
  int side;           // runtime side when SIDE_T < 0 (warp-uniform)
  float* dump_h;      // DUMP (test hook morea_sample_map): per-voxel h and fg of this side
  unsigned char* dump_fg;
  int qoff;           // row hulls of this side at the item's radius: V.qhull[0] + qoff
                      // + z ny + y; -1 when there are none (empty-space skip off)
  // CLAMP: some position of the item may leave the range the gather covers
  // exactly, apply the O5 clamp (a separate instantiation: no predicated clamp
  // instructions in the common loop)

  // per-side data selected by a warp-uniform branch on compile-time parameter
  // offsets, so texture handles stay in uniform registers
  __device__ __forceinline__ const float* vol(int s) const { return s == 0 ? V.I[0] : V.I[1]; }

  // the 8 corners (i0 .. i0+1)^3: two 2x2 texture gathers (tld4) or 8 loads
  __device__ __forceinline__ void gather(const float* __restrict__ vol, unsigned long long tex,
                                         float u, float v, int base, float c[8]) const {
    if (TEX) {
      const float4 g0 = tex2Dgather<float4>((cudaTextureObject_t)tex, u, v, 0);
      const float4 g1 = tex2Dgather<float4>((cudaTextureObject_t)tex, u, v + V.fnyp, 0);
      // gather order: (x0,y1) (x1,y1) (x1,y0) (x0,y0)
      c[0] = g0.w; c[1] = g0.z; c[2] = g0.x; c[3] = g0.y;
      c[4] = g1.w; c[5] = g1.z; c[6] = g1.x; c[7] = g1.y;
    } else {
      const int sy = V.nx, sz = V.nx * V.ny;
      c[0] = __ldg(&vol[base]); c[1] = __ldg(&vol[base + 1]);
      c[2] = __ldg(&vol[base + sy]); c[3] = __ldg(&vol[base + sy + 1]);
      c[4] = __ldg(&vol[base + sz]); c[5] = __ldg(&vol[base + sz + 1]);
      c[6] = __ldg(&vol[base + sz + sy]); c[7] = __ldg(&vol[base + sz + sy + 1]);
    }
  }

  __device__ __forceinline__ static float tri(const float c[8], float fx, float fy, float fz,
                                              float gx, float gy, float gz) {
    return plerp(plerp(plerp(c[0], c[1], fx, gx), plerp(c[2], c[3], fx, gx), fy, gy),
                 plerp(plerp(c[4], c[5], fx, gx), plerp(c[6], c[7], fx, gx), fy, gy), fz, gz);
  }

  // tld4 pair (slices i0_z and i0_z + 1); u carries the volume's x offset
  __device__ __forceinline__ void gather_tex(float u, float v, float c[8]) const {
    const float4 g0 = tex2Dgather<float4>((cudaTextureObject_t)V.texI, u, v, 0);
    const float4 g1 = tex2Dgather<float4>((cudaTextureObject_t)V.texI, u, v + V.fnyp, 0);
    // gather order: (x0,y1) (x1,y1) (x1,y0) (x0,y0)
    c[0] = g0.w; c[1] = g0.z; c[2] = g0.x; c[3] = g0.y;
    c[4] = g1.w; c[5] = g1.z; c[6] = g1.x; c[7] = g1.y;
  }

  // guidance term of one band entry (a6, O8): pair i of the side-s sample with
  // own-record index lin = s V + q, mapped to texel u, v and weights fx, fy, fz
  __device__ __forceinline__ void entry(float u, float v, float fx, float fy, float fz, int lin,
                                        int i, int s) {
    const int o = 1 - s;
    // map i of side s at voxel q = lin - s V: element i V + q < K V <= 8 * 768^3 < 2^32
    // (morea_load_images bounds), so the index is computed in 32-bit unsigned
    // arithmetic (mod 2^32, exact)
    const unsigned di = (unsigned)(i - s) * (unsigned)V.V + (unsigned)lin;
    const float d = __ldg(&(s == 0 ? V.dmap[0] : V.dmap[1])[di]);
    float e[8];
    if (TEX) {
      // u = i0_x + uoff0 + o fnxp (texel of I_o); map (o, i) is volume o K + i of texM
      const float uu = fmaf((float)(o * (V.K - 1) + i), V.fnxp, u);
      const float4 g0 = tex2Dgather<float4>((cudaTextureObject_t)V.texM, uu, v, 0);
      const float4 g1 = tex2Dgather<float4>((cudaTextureObject_t)V.texM, uu, v + V.fnyp, 0);
      e[0] = g0.w; e[1] = g0.z; e[2] = g0.x; e[3] = g0.y;
      e[4] = g1.w; e[5] = g1.z; e[6] = g1.x; e[7] = g1.y;
    } else {
      const int base = (int)(v - 1.0f) * V.nx + (int)(u - 1.0f);
      gather((o == 0 ? V.dmap[0] : V.dmap[1]) + (long long)i * V.V, 0ull, 0.f, 0.f, base, e);
    }
    const float Dp = tri(e, fx, fy, fz, 1.f - fx, 1.f - fy, 1.f - fz);
    const float dd = d - Dp;
    // O8: w_i (r - d)/r (d - D'(x))^2, only where d < r (band bit).  r - d as
    // (r_f - d) + (r - r_f): exact first difference for d >= r_f / 2, so the
    // relative error of the small differences near the band edge stays at ulp
    // level.  Term in fp32, partial sums in fp32 (flushed with h), sum in fp64.
    const float rd = (V.rf - d) + V.rlo;
    acc.gf += V.wf[s][i] * rd * (dd * dd);
  }

  // Band entries of this step's samples, one round per set bit, go to the
  // per-warp queue, evaluated 32 at a time (acc.qn: queued count, warp-uniform).
  __device__ __forceinline__ void enqueue(unsigned bm, unsigned take, int lin, float u, float v, float fx,
                                          float fy, float fz, int s) {
    // take: the ballot of bm != 0 (non-zero: the caller's test)
    const int lane = threadIdx.x & 31;
    do {
      {
        // computed by every lane, stored by lanes with a bit: predicated stores,
        // no divergent branch (no convergence barrier per round)
        const int i = __ffs(bm) - 1;
        const int pos = acc.qn + __popc(take & ((1u << lane) - 1u));
        MOREA_CHECK(pos < kQueueCap);
        const unsigned qa_addr = (unsigned)__cvta_generic_to_shared(&S.qa[pos]);
        const unsigned qb_addr = (unsigned)__cvta_generic_to_shared(&S.qb[pos]);
        const unsigned qi_addr = (unsigned)__cvta_generic_to_shared(&S.qi[pos]);
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.u32 p, %0, 0;\n"
            " @p st.shared.v4.f32 [%1], {%4, %5, %6, %7};\n"
            " @p st.shared.v2.b32 [%2], {%8, %9};\n"
            " @p st.shared.u8 [%3], %10;\n}"
            :
            : "r"(bm), "r"(qa_addr), "r"(qb_addr), "r"(qi_addr), "f"(u), "f"(v), "f"(fx), "f"(fy),
              "r"(__float_as_int(fz)), "r"(lin), "r"(i)
            : "memory");
        bm &= bm - 1u;
      }
      acc.qn += __popc(take);
      if (__all_sync(FULLMASK, acc.qn >= 32)) {  // warp-uniform (VOTE): no BSSY
        acc.qn -= 32;
        if (lane == 0) S.stat[1] += 32;  // band entries: each queued entry is evaluated once
        __syncwarp();
        const float4 ea = S.qa[acc.qn + lane];
        const int2 eb = S.qb[acc.qn + lane];
        entry(ea.x, ea.y, ea.z, ea.w, __int_as_float(eb.x), eb.y, (int)S.qi[acc.qn + lane], s);
        __syncwarp();
      }
      take = __ballot_sync(FULLMASK, bm != 0u);
    } while (take);
  }

  __device__ __forceinline__ void count_only(int t) { acc.n += t; }

  // quiet rows (raster): the side's row hulls at the item's radius R (SideRec flags)
  static constexpr bool kQuiet = true;
  __device__ __forceinline__ int quiet_off() const { return qoff; }
  __device__ __forceinline__ unsigned quiet_hull(int idx) const {
    // one 32-bit load of the packed short2 (first, last)
    return __ldg(reinterpret_cast<const unsigned*>(V.qhull[0]) + idx);  // qoff carries the side
  }
  // samples of a chunk's quiet rows (profiling; lane 0, per-warp shared counter)
  __device__ __forceinline__ void count_quiet(int n) { S.swept += (unsigned)n; }
  __device__ __forceinline__ void quiet_row(int q0, int n) {
    if (DUMP)
      for (int i = 0; i < n; i++) {
        dump_h[q0 + i] = 0.f;
        dump_fg[q0 + i] = 0;
      }
  }

  // the fp32 partial sums are flushed into the fp64 lane sums once at least 16 steps
  // have been added since the last flush (so at most 15 + 32 = 47 steps per fp32 sum)
  __device__ __forceinline__ void steps_done(int n) {
    acc.ns += n;
    if (acc.ns >= 16) {
      flush_h();
      acc.ns = 0;
    }
  }

  __device__ __forceinline__ void flush_h() {
    const double h = acc.hg[0], g = acc.hg[1];
    acc.hg[0] = h + (double)acc.hf;
    acc.hf = 0.f;
    acc.hg[1] = g + (double)acc.gf;
    acc.gf = 0.f;
  }

  // evaluate what is left in the queue (end of a side)
  __device__ __forceinline__ void drain(int s) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    if (lane == 0) S.stat[1] += (unsigned long long)acc.qn;
    if (lane < acc.qn) {
      const float4 ea = S.qa[lane];
      const int2 eb = S.qb[lane];
      entry(ea.x, ea.y, ea.z, ea.w, __int_as_float(eb.x), eb.y, (int)S.qi[lane], s);
    }
    __syncwarp();
    acc.qn = 0;
    flush_h();
  }

  __device__ __forceinline__ void sample(const int4& ra, const float4& rb, int k, bool valid) {
    const int SIDE = SIDE_T >= 0 ? SIDE_T : side;
    const int OTH = 1 - SIDE;
    const int nx = V.nx, ny = V.ny, nz = V.nz;
    const int lin = ra.y + k;
    MOREA_CHECK(!valid || (lin >= (long long)SIDE * V.V && lin < (long long)(SIDE + 1) * V.V));
    const uint2 own = __ldg(&V.own[0][lin]);  // lin = SIDE V + q
    const float a = __uint_as_float(own.x);
    const unsigned bm = valid ? own.y : 0u;  // the band byte (k_own_records: upper bits 0)
    const float kf = (float)k;
    const float4 s0 = sc0;
    const float dx = fmaf(s0.x, kf, __int_as_float(ra.z)), dy = fmaf(s0.y, kf, __int_as_float(ra.w)),
                dz = fmaf(s0.z, kf, rb.x);
    const float flx = floorf(dx), fly = floorf(dy), flz = floorf(dz);
    float fx = dx - flx, fy = dy - fly, fz = dz - flz;
    const float4 s1 = sc1;
    const bool amb = (fabsf(fx - 0.5f) > s0.w) | (fabsf(fy - 0.5f) > s1.x) | (fabsf(fz - 0.5f) > s1.y);
    // lattice corner i0 as exact floats (< 2^24)
    float ix = rb.y + kf + flx, iy = rb.z + fly, iz = rb.w + flz;
    if (CLAMP) {
      // O5 clamp: x <= 0 -> (0, f = 0), x >= n-1 -> (n-2, f = 1)
      fx = ix < 0.f ? 0.f : (ix > V.fnx2 ? 1.f : fx);
      fy = iy < 0.f ? 0.f : (iy > V.fny2 ? 1.f : fy);
      fz = iz < 0.f ? 0.f : (iz > V.fnz2 ? 1.f : fz);
      ix = fminf(fmaxf(ix, 0.f), V.fnx2);
      iy = fminf(fmaxf(iy, 0.f), V.fny2);
      iz = fminf(fmaxf(iz, 0.f), V.fnz2);
    }
    const float gx = 1.f - fx, gy = 1.f - fy, gz = 1.f - fz;
    // gather coordinates of corner i0 (Volumes::fnxp; exact floats)
    const float u = ix + s1.z, v = fmaf(iz, V.fnyp, iy) + V.voff;
    const int base = TEX ? 0 : ((int)iz * ny + (int)iy) * nx + (int)ix;
    float c[8];
    // the footprint lies inside the padded layout (positions in (-1, n) or clamped):
    // gather at integer (u, v) reads texel columns u-1, u and rows v-1, v (+ fnyp)
    MOREA_CHECK(!TEX || !valid || (u >= 1.f && u <= 2.f * V.fnxp - 1.f));
    MOREA_CHECK(!TEX || !valid || (v >= 1.f && v + V.fnyp <= V.fnyp * (float)(nz + 2) - 1.f));
    MOREA_CHECK(TEX || !valid || (base >= 0 && (long long)base + (long long)nx * ny + nx + 1 < V.V));
    if (TEX) gather_tex(u, v, c);
    else gather(vol(OTH), 0ull, u, v, base, c);
    const float b = tri(c, fx, fy, fz, gx, gy, gz);
    bool fg = b > 0.f;
    // warp-uniform branch around the rare exact path: no convergence barrier
    // (BSSY/BMOV/BSYNC) in the common path (measured 2% faster)
    if (__any_sync(FULLMASK, amb))
      fg = exact_fg_if(amb, fg, R, (int)rb.y + k, (int)rb.z, (int)rb.w, dx, dy, dz, vol(OTH), nx, ny, nz);
    // h of PAPER.md §4.1.2 (L318-322) with the exact case split (O6)
    float h;
    if (a > 0.f && fg) {
      const float t = a - b;
      h = t * t;
    } else {
      h = (a == 0.f && !fg) ? 0.f : 1.f;
    }
    // fp32 partial sum over at most 47 steps; raster() flushes it into the fp64
    // lane sum (steps_done / flush_h) once 16 or more steps accumulated
    acc.hf += valid ? h : 0.f;
    if (DUMP && valid) {  // the values just computed, at voxel q = lin - SIDE V
      const long long q = (long long)lin - (long long)SIDE * V.V;
      dump_h[q] = h;
      dump_fg[q] = fg ? 1 : 0;
    }
    // a6: band entries go to the per-warp queue, evaluated 32 at a time
    const unsigned take = __ballot_sync(FULLMASK, bm != 0u);
    if (take) enqueue(bm, take, lin, u, v, fx, fy, fz, SIDE);
  }
};


// Debug builds: the BlockQueue hands out every item exactly once.  Each processed
// item is counted; the last block to finish checks the count against n_items (a
// lost or a duplicated claim fails the check).
__device__ __forceinline__ void debug_count_item(const EvalArgs& A) {
#ifdef MOREA_DEBUG_CHECKS
  atomicAdd(&A.counter[1], 1ull);
#endif
}
__device__ __forceinline__ void debug_check_items(const EvalArgs& A, long long n_items) {
#ifdef MOREA_DEBUG_CHECKS
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long done = atomicAdd(&A.counter[2], 1ull);
    if (done == gridDim.x - 1) {
      __threadfence();
      MOREA_CHECK(atomicAdd(&A.counter[1], 0ull) == (unsigned long long)n_items);
    }
  }
#endif
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
  return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
  return v;
}

// warp-cooperative copy of one SideRec into shared memory
__device__ __forceinline__ void load_rec(WarpSmem& S, const SideRec* src, int lane) {
  constexpr int kVec = (int)(sizeof(SideRec) / 16);
  __syncwarp();
  if (lane < kVec)
    reinterpret_cast<int4*>(&S.R)[lane] = __ldg(reinterpret_cast<const int4*>(src) + lane);
  __syncwarp();
  // edge table for slice_y_range: lane e < 6 takes edge (0,1) (0,2) (0,3) (1,2) (1,3) (2,3)
  if (lane < 6) {
    const int i = lane < 3 ? 0 : (lane < 5 ? 1 : 2);
    const int j = lane < 3 ? lane + 1 : (lane < 5 ? lane - 1 : 3);
    float zi = S.R.vz[i], zj = S.R.vz[j], yi = S.R.vy[i], yj = S.R.vy[j];
    if (zj < zi) {
      const float tz = zi, ty = yi;
      zi = zj; yi = yj; zj = tz; yj = ty;
    }
    const bool flat = !(zj > zi);
    S.edge[lane] = make_float4(zi, zj, yi, flat ? 0.f : (yj - yi) / (zj - zi));
    S.edge_y1[lane] = flat ? yj : __int_as_float(0x7fffffff);  // NaN: no second end
  }
  __syncwarp();
}

template <bool TEX, int SIDE_T, bool DUMP>
__device__ __forceinline__ void raster_side(const Volumes& V, WarpSmem& S, int lane, Acc& acc,
                                            int side, float* dump_h, unsigned char* dump_fg) {
  const SideRec& R = S.R;
  if (lane == 0) {
    S.sc0 = make_float4(R.A[0][0], R.A[1][0], R.A[2][0], 0.5f - R.eps[0]);
    // gather x of corner i0: I_o is volume o of texI (TEX), else a plain index + 1
    const float uoff = TEX ? fmaf((float)(1 - (SIDE_T >= 0 ? SIDE_T : side)), V.fnxp, V.uoff0) : 1.0f;
    S.sc1 = make_float4(0.5f - R.eps[1], 0.5f - R.eps[2], uoff, 0.f);
  }
  __syncwarp();
  // O5 clamp only where a position can leave the range the gather covers exactly:
  // [0, n-1) for plain loads, (-1, n) on the edge-padded textures (warp-uniform)
  const int loff = (SIDE_T >= 0 ? SIDE_T : side) * (int)V.V;
  const int qR = (R.flags >> 8) & 0xff;  // empty-space radius of the item (k_setup)
  // row hulls of this side at radius qR, as an offset from V.qhull[0] (the two sides'
  // tables are contiguous: qhull[1] = qhull[0] + nR ny nz, morea_api.cu)
  const int nR = kQuietRmax - kQuietRmin + 1;
  const int qoff = (V.qhull[0] && qR <= kQuietRmax)
                       ? ((SIDE_T >= 0 ? SIDE_T : side) * nR + (qR - kQuietRmin)) * V.ny * V.nz
                       : -1;
  if ((R.flags & ((TEX && kTexPad) ? 8 : 2)) == 0) {
    Sample<TEX, SIDE_T, true, DUMP> f{V, R, S, S.sc0, S.sc1, acc, side, dump_h, dump_fg, qoff};
    raster(R, V.nx, V.ny, loff, S, lane, f);
    f.drain(SIDE_T >= 0 ? SIDE_T : side);
  } else {
    Sample<TEX, SIDE_T, false, DUMP> f{V, R, S, S.sc0, S.sc1, acc, side, dump_h, dump_fg, qoff};
    raster(R, V.nx, V.ny, loff, S, lane, f);
    f.drain(SIDE_T >= 0 ? SIDE_T : side);
  }
}


// Block-local item dispenser for the one-block-per-SM kernels: warps take
// consecutive items of the block's current chunk (the same tet for consecutive
// solutions, so footprints still share the SM's L1) without a block barrier per
// claim.  Lane 0 of one warp at a time holds a shared-memory lock; the warp that
// finds the chunk empty claims the next one from the global queue.  Items come
// out in increasing order, so a warp that sees item >= n_items can stop.
// (Measured against the block-barrier claim: k_raster C4 full 48.4 -> 47.4 ms.)
struct BlockQueue {
  unsigned long long next, end;
  int lock;
  __device__ __forceinline__ void init() {  // all threads of the block; ends with a barrier
    if (threadIdx.x == 0) {
      next = end = 0ull;
      lock = 0;
    }
    __syncthreads();
  }
  // chunk: at most max_chunk items per global claim, fewer when the launch has
  // under `spread` claims per block (the largest-first order puts the big tets
  // in the first chunks; larger chunks measured slower at C4).  Computed at
  // refill time only (no register held across the item loop).
  __device__ __forceinline__ unsigned long long claim(unsigned long long* counter, int lane,
                                                      long long n_items, int max_chunk, int spread) {
    unsigned long long n = 0;
    if (lane == 0) {
      while (atomicCAS(&lock, 0, 1) != 0) __nanosleep(20);
      __threadfence_block();
      volatile unsigned long long* vn = &next;
      volatile unsigned long long* ve = &end;
      n = *vn;
      if (n >= *ve) {
        const unsigned long long chunk = (unsigned long long)max(
            1LL, min((long long)max_chunk, n_items / ((long long)gridDim.x * spread)));
        n = atomicAdd(counter, chunk);
        *ve = n + chunk;
      }
      *vn = n + 1;
      __threadfence_block();
      atomicExch(&lock, 0);
    }
    return __shfl_sync(FULLMASK, n, 0);
  }
};

// ---------------------------------------------------------------------------
// k_raster: persistent warps over the item queue (a4 + a5 + a6 + per-tet a7).
// ---------------------------------------------------------------------------
// one block per SM: its warps take consecutive items (the same tet for
// consecutive solutions) together, so their footprints share the SM's L1
constexpr int kRasterBlockWarps = MOREA_SM_BLOCK;
constexpr int kRasterBlockThreads = 32 * kRasterBlockWarps;
#define RASTER_BOUNDS __launch_bounds__(kRasterBlockThreads, 1)

template <bool TEX, bool DUMP>
__global__ void RASTER_BOUNDS k_raster(const EvalArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmem* smem = reinterpret_cast<WarpSmem*>(smem_raw);
  __shared__ BlockQueue bq;
  bq.init();
  // warp index and lane through volatile asm: kept in registers instead of being
  // re-derived from special registers at every use
  int warp, lane;
  asm volatile("shr.u32 %0, %1, 5;" : "=r"(warp) : "r"(threadIdx.x));
  asm volatile("and.b32 %0, %1, 31;" : "=r"(lane) : "r"(threadIdx.x));
  WarpSmem& S = smem[warp];
  const long long per_v = (long long)A.n_entries * A.P;
  const long long n_items = per_v * A.n_raster_versions;
  if (lane == 0) {
    S.stat[0] = S.stat[1] = S.stat[2] = S.stat[3] = 0ull;
    S.swept = 0u;
  }
  while (true) {
    unsigned long long item = 0;
    item = bq.claim(A.counter, lane, n_items, MOREA_CLAIM_CHUNK, MOREA_CLAIM_SPREAD);
    if ((long long)item >= n_items) break;
    const int v = (int)(item / (unsigned long long)per_v);
    const long long rem = (long long)item - (long long)v * per_v;
    const int es = (int)(rem / A.P);
    const int sol = (int)(rem - (long long)es * A.P);
    const int e = A.sched[es];
    MOREA_CHECK(e >= 0 && e < A.n_entries && v < A.n_raster_versions);
    const long long i = ((long long)v * A.n_entries + e) * A.P + sol;
    double hg_local[2] = {0.0, 0.0};
    Acc acc{hg_local, 0.f, 0.f, 0, 0, 0};
    int n_side0 = 0;
#pragma unroll 1
    for (int side = 0; side < 2; side++) {
      if (DUMP && side != A.dump_side) continue;
      load_rec(S, &A.geom[2 * i + side], lane);
      if (S.R.flags & 1) raster_side<TEX, -1, DUMP>(A.vol, S, lane, acc, side, A.dump_h, A.dump_fg);
      if (side == 0) n_side0 = acc.n;
    }
    HGN out;
    out.h = warp_sum_d(acc.hg[0] + (double)acc.hf);
    out.g = warp_sum_d(acc.hg[1]);
    out.n = warp_sum_i(acc.n);
    out.n0 = warp_sum_i(n_side0);
    if (lane == 0) {
      A.hgn[i] = out;
      S.stat[0] += out.n;
      S.stat[2] += 1;
      S.stat[3] += (unsigned long long)(out.n - (long long)S.swept);  // quiet = samples - swept
      S.swept = 0u;
      debug_count_item(A);
    }
  }
  debug_check_items(A, n_items);
  if (lane == 0 && A.stats) {
    atomicAdd(&A.stats[0], S.stat[0]);
    atomicAdd(&A.stats[1], S.stat[1]);
    atomicAdd(&A.stats[2], S.stat[2]);
    atomicAdd(&A.stats[3], S.stat[3]);
  }
}

constexpr size_t kRasterDynSmem = MOREA_SM_BLOCK ? sizeof(WarpSmem) * kRasterBlockWarps : 0;
// shared memory decides the L1/shared carve-out of the SM (steps 100, 132, ...
// KB, 1 KB per block reserved by the system): at <= 99 KB the carve-out is
// 100 KB and the texture/L1 cache keeps 156 KB (measured: 8 KB more shared
// memory, crossing a step, costs 2.3%)
static_assert(!MOREA_SM_BLOCK || kRasterDynSmem + 1024 + 64 <= 100 * 1024,
              "k_raster shared memory above the 100 KB carve-out step");

int raster_blocks_per_sm(bool tex) {
  if (kRasterDynSmem) {
    cudaFuncSetAttribute(k_raster<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRasterDynSmem);
    cudaFuncSetAttribute(k_raster<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRasterDynSmem);
    cudaFuncSetAttribute(k_raster<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRasterDynSmem);
    cudaFuncSetAttribute(k_raster<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRasterDynSmem);
  }
  int nb = 0;
  cudaError_t e = tex ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_raster<true, false>,
                                                                      kRasterBlockThreads, kRasterDynSmem)
                      : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_raster<false, false>,
                                                                      kRasterBlockThreads, kRasterDynSmem);
  if (e != cudaSuccess) return 1;
  return nb > 0 ? nb : 1;
}

int raster_block_warps() { return kRasterBlockWarps; }

cudaError_t launch_raster(const EvalArgs& a, int grid, cudaStream_t s) {
  if (a.dump_h) {  // test hook morea_sample_map
    if (a.vol.use_tex) k_raster<true, true><<<grid, kRasterBlockThreads, kRasterDynSmem, s>>>(a);
    else k_raster<false, true><<<grid, kRasterBlockThreads, kRasterDynSmem, s>>>(a);
  } else {
    if (a.vol.use_tex) k_raster<true, false><<<grid, kRasterBlockThreads, kRasterDynSmem, s>>>(a);
    else k_raster<false, false><<<grid, kRasterBlockThreads, kRasterDynSmem, s>>>(a);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// a7 / a8: per (solution, group) reduction in a fixed order (warp per output),
// objectives, flags, and the per-tet cache outputs.
// ---------------------------------------------------------------------------
__global__ void k_reduce(const EvalArgs A, int G, const int* __restrict__ group_off,
                         const morea_acc* __restrict__ base_acc, const double* __restrict__ cache_in,
                         double* __restrict__ cache_out, const int* __restrict__ changed,
                         const int* __restrict__ grp_off, double* __restrict__ obj,
                         morea_acc* __restrict__ acc) {
  const int lane = threadIdx.x & 31;
  const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int P = A.P;
  if (wid >= (long long)P * G) return;
  const int sol = (int)(wid / G), g = (int)(wid % G);
  const int T = A.mesh.T, N = A.mesh.N;
  const long long per_v = (long long)A.n_entries * P;
  double h = 0.0, gs = 0.0, m = 0.0, sev = 0.0;
  long long n = 0, n0 = 0;
  int folds = 0, dom = 0;
  for (int e = group_off[g] + lane; e < group_off[g + 1]; e += 32) {
    const long long i0 = (long long)e * P + sol;
    const Scal s0 = A.scal[i0];
    const HGN r0 = A.hgn[i0];
    const int tet = A.canon_tet ? A.canon_tet[e] : e;
    dom |= s0.flags & 1;
    if (!A.partial) {
      h += r0.h; gs += r0.g; m += s0.m; sev += s0.sev; n += r0.n; n0 += r0.n0; folds += s0.folds;
      if (cache_out) {
        double* c = cache_out + ((long long)sol * T + tet) * 4;
        c[0] = r0.h; c[1] = r0.g; c[2] = (double)r0.n; c[3] = s0.m;
      }
    } else {
      const Scal s1 = A.scal[i0 + per_v];
      double oh, og;
      long long on;
      if (cache_in) {
        const double* c = cache_in + ((long long)sol * T + tet) * 4;
        oh = c[0]; og = c[1]; on = (long long)c[2];
      } else {
        const HGN r1 = A.hgn[i0 + per_v];
        oh = r1.h; og = r1.g; on = r1.n;
      }
      h += r0.h - oh; gs += r0.g - og; m += s0.m - s1.m; sev += s0.sev - s1.sev;
      n += r0.n - on; folds += s0.folds - s1.folds;
      if (cache_out) {
        double* c = cache_out + ((long long)sol * A.n_entries + e) * 4;
        c[0] = r0.h; c[1] = r0.g; c[2] = (double)r0.n; c[3] = s0.m;
      }
    }
  }
  // domain check of the points that define this output (all points for a full
  // evaluation, the new values of S_g for a partial one)
  if (!A.partial) {
    for (int j = lane; j < N; j += 32)
      for (int c = 0; c < 6; c++) {
        const i64 q = canon_q(A.mesh.base[3 * j + (c % 3)], A.offsets[((long long)sol * N + j) * 6 + c]);
        if (q < kQLo || q >= kQHi) dom = 1;
      }
  } else {
    for (int i = grp_off[g] + lane; i < grp_off[g + 1]; i += 32) {
      const int j = changed[i];
      for (int c = 0; c < 6; c++) {
        const i64 q = canon_q(A.mesh.base[3 * j + (c % 3)], A.new_vals[((long long)sol * A.S_total + i) * 6 + c]);
        if (q < kQLo || q >= kQHi) dom = 1;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    h += __shfl_xor_sync(FULLMASK, h, o);
    gs += __shfl_xor_sync(FULLMASK, gs, o);
    m += __shfl_xor_sync(FULLMASK, m, o);
    sev += __shfl_xor_sync(FULLMASK, sev, o);
    n += __shfl_xor_sync(FULLMASK, n, o);
    n0 += __shfl_xor_sync(FULLMASK, n0, o);
    folds += __shfl_xor_sync(FULLMASK, folds, o);
    dom |= __shfl_xor_sync(FULLMASK, dom, o);
  }
  if (lane != 0) return;
  morea_acc out;
  if (A.partial) {
    const morea_acc b = base_acc[sol];
    out.h_sum = b.h_sum + h;
    out.g_sum = b.g_sum + gs;
    out.m_sum = b.m_sum + m;
    out.severity = b.severity + sev;
    out.n_samples = b.n_samples + n;
    out.folds = b.folds + folds;
    out.flags = (b.flags & MOREA_F_DOMAIN) | (dom ? MOREA_F_DOMAIN : 0);
  } else {
    out.h_sum = h; out.g_sum = gs; out.m_sum = m; out.severity = sev;
    out.n_samples = n; out.folds = folds;
    out.flags = dom ? MOREA_F_DOMAIN : 0;
    if (A.expect[0] >= 0 && !dom && (n0 != A.expect[0] || n - n0 != A.expect[1]))
      out.flags |= MOREA_F_COVERAGE;  // row a9 coverage check
  }
  if (out.n_samples == 0) out.flags |= MOREA_F_EMPTY;
  const long long o = (long long)sol * G + g;
  if (acc) acc[o] = out;
  if (obj) {
    if (out.flags & (MOREA_F_DOMAIN | MOREA_F_EMPTY)) {
      obj[3 * o] = obj[3 * o + 1] = obj[3 * o + 2] = __longlong_as_double(0x7ff8000000000000LL);
    } else {
      obj[3 * o + 0] = out.m_sum / (10.0 * (double)T);     // L258
      obj[3 * o + 1] = out.h_sum / (double)out.n_samples;  // L317
      obj[3 * o + 2] = out.g_sum / (double)out.n_samples;  // L339
    }
  }
}

cudaError_t launch_reduce(const EvalArgs& a, int G, const int* group_off, const void* base_acc,
                          const double* cache_in, double* cache_out, const int* changed,
                          const int* grp_off, double* obj, void* acc, cudaStream_t s) {
  const long long warps = (long long)a.P * G;
  if (warps == 0) return cudaSuccess;
  const int threads = 256;
  const long long blocks = (warps * 32 + threads - 1) / threads;
  k_reduce<<<(unsigned)blocks, threads, 0, s>>>(a, G, group_off, (const morea_acc*)base_acc, cache_in,
                                                cache_out, changed, grp_off, obj, (morea_acc*)acc);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// a9: fold check only.  Warp per solution, lanes stride the tets in a fixed
// order, fixed shuffle tree => deterministic.
// ---------------------------------------------------------------------------
__global__ void k_check_folds(MeshDev M, double sp0, double sp1, double sp2, int P,
                              const float* __restrict__ offsets, int* __restrict__ count,
                              double* __restrict__ sev_out, unsigned char* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int sol = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (sol >= P) return;
  int cnt = 0;
  double sev = 0.0;
  for (int t = lane; t < M.T; t += 32) {
    const int4 tv = M.tets[t];
    const int vid[4] = {tv.x, tv.y, tv.z, tv.w};
    int Q[2][4][3];
    bool ok = true;
    for (int k = 0; k < 4; k++) {
      const float2* o = reinterpret_cast<const float2*>(offsets + ((long long)sol * M.N + vid[k]) * 6);
      const float2 o01 = __ldg(o), o23 = __ldg(o + 1), o45 = __ldg(o + 2);  // 24 contiguous bytes
      const float oo[6] = {o01.x, o01.y, o23.x, o23.y, o45.x, o45.y};
      for (int a = 0; a < 3; a++)
        for (int s = 0; s < 2; s++) {
          const i64 q = canon_q(M.base[3 * vid[k] + a], oo[3 * s + a]);
          ok = ok && q >= kQLo && q < kQHi;
          Q[s][k][a] = (int)q;
        }
    }
    for (int s = 0; s < 2; s++) {
      int f = 0;
      if (ok) {
        const i64 det = det3(Q[s]);
        const int sg = (det > 0) - (det < 0);
        if (sg != M.ref[t]) {
          f = 1;
          cnt += 1;
          sev += (double)(det < 0 ? -det : det) / (6.0 * 1073741824.0) * sp0 * sp1 * sp2;
        }
      }
      if (flags) flags[((long long)sol * 2 + s) * M.T + t] = (unsigned char)f;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    cnt += __shfl_xor_sync(FULLMASK, cnt, o);
    sev += __shfl_xor_sync(FULLMASK, sev, o);
  }
  if (lane == 0) {
    if (count) count[sol] = cnt;
    if (sev_out) sev_out[sol] = sev;
  }
}

cudaError_t launch_check_folds(const MeshDev& m, const double sp[3], int P, const float* offsets,
                               int* count, double* sev, unsigned char* flags, cudaStream_t s) {
  const int threads = 256;
  const long long blocks = ((long long)P * 32 + threads - 1) / threads;
  k_check_folds<<<(unsigned)blocks, threads, 0, s>>>(m, sp[0], sp[1], sp[2], P, offsets, count, sev,
                                                     flags);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Owner-map test hook: the same SideRec + rasterizer, one warp per tet.
// ---------------------------------------------------------------------------
struct OwnerSample {
  int* owner;
  int tet;
  static constexpr bool kQuiet = false;
  __device__ __forceinline__ int quiet_off() const { return -1; }
  __device__ __forceinline__ unsigned quiet_hull(int) const { return 0xffff0000u; }
  __device__ __forceinline__ void count_quiet(int) {}
  __device__ __forceinline__ void quiet_row(int, int) {}
  __device__ __forceinline__ void steps_done(int) {}
  __device__ __forceinline__ void flush_h() {}
  __device__ __forceinline__ void count_only(int) {}
  __device__ __forceinline__ void sample(const int4& ra, const float4&, int k, bool valid) {
    if (!valid) return;
    const int lin = ra.y + k;
    const int old = atomicCAS(&owner[lin], -1, tet);
    if (old != -1) atomicExch(&owner[lin], -2);
  }
};

__global__ void __launch_bounds__(kRasterThreads) k_owner_map(const EvalArgs A, int side,
                                                              int* __restrict__ owner) {
  __shared__ WarpSmem smem[kWarpsPerBlock];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tet = blockIdx.x * kWarpsPerBlock + warp;
  if (tet >= A.mesh.T) return;
  WarpSmem& S = smem[warp];
  load_rec(S, &A.geom[2 * (long long)tet + side], lane);
  if (!(S.R.flags & 1)) return;
  OwnerSample f{owner, tet};
  raster(S.R, A.vol.nx, A.vol.ny, 0, S, lane, f);
}

__global__ void k_fill_int(int* p, long long n, int v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_fill_dump(float* h, unsigned char* fg, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    h[i] = __int_as_float(0x7fc00000);
    fg[i] = 255;
  }
}

cudaError_t launch_fill(float* h, unsigned char* fg, long long V, cudaStream_t s) {
  k_fill_dump<<<1024, 256, 0, s>>>(h, fg, V);
  return cudaGetLastError();
}

cudaError_t launch_owner_map(const EvalArgs& a, int side, int* owner, cudaStream_t s) {
  k_fill_int<<<1024, 256, 0, s>>>(owner, a.vol.V, -1);
  cudaError_t e = launch_setup(a, s);
  if (e != cudaSuccess) return e;
  const int blocks = (a.mesh.T + kWarpsPerBlock - 1) / kWarpsPerBlock;
  k_owner_map<<<blocks, kRasterThreads, 0, s>>>(a, side, owner);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// a0: load-time work.
// ---------------------------------------------------------------------------
__global__ void k_validate_volume(const float* __restrict__ I, long long V, int* bad) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < V;
       i += (long long)gridDim.x * blockDim.x) {
    const float v = I[i];
    // finite, >= 0, and either exactly 0 (background) or >= 2^-40
    if (!(v >= 0.0f) || isinf(v) || (v > 0.0f && v < 9.094947017729282e-13f)) atomicOr(bad, 1);
  }
}

cudaError_t launch_validate_volume(const float* I, long long V, int* bad, cudaStream_t s) {
  k_validate_volume<<<1024, 256, 0, s>>>(I, V, bad);
  return cudaGetLastError();
}

// Exact nearest-point distance (O8): min over ALL points of the pair of
// ((q-c) s)^2 in fp64 with the operation order ((dx^2 + dy^2) + dz^2) and no
// contraction, sqrt, rounded once to fp32.  Points are staged through shared
// memory; one thread per voxel.
constexpr int kDistTile = 512;
__global__ void __launch_bounds__(256) k_distance_maps(const float* __restrict__ pts,
                                                       const long long* __restrict__ off, int K,
                                                       int nx, int ny, int nz, double s0, double s1,
                                                       double s2, float* __restrict__ dmap) {
  __shared__ float sp[kDistTile * 3];
  const long long V = (long long)nx * ny * nz;
  const int i = blockIdx.y;  // pair
  const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = v < V;
  const int x = active ? (int)(v % nx) : 0;
  const int y = active ? (int)((v / nx) % ny) : 0;
  const int z = active ? (int)(v / ((long long)nx * ny)) : 0;
  const double qx = x, qy = y, qz = z;
  double best = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  const long long c0 = off[i], c1 = off[i + 1];
  for (long long t0 = c0; t0 < c1; t0 += kDistTile) {
    const int nt = (int)min((long long)kDistTile, c1 - t0);
    __syncthreads();
    for (int t = threadIdx.x; t < nt * 3; t += blockDim.x) sp[t] = pts[t0 * 3 + t];
    __syncthreads();
    for (int t = 0; t < nt; t++) {
      const double dx = __dmul_rn(__dsub_rn(qx, (double)sp[3 * t + 0]), s0);
      const double dy = __dmul_rn(__dsub_rn(qy, (double)sp[3 * t + 1]), s1);
      const double dz = __dmul_rn(__dsub_rn(qz, (double)sp[3 * t + 2]), s2);
      const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      best = fmin(best, d2);
    }
  }
  if (active) dmap[(long long)i * V + v] = __double2float_rn(__dsqrt_rn(best));
}

cudaError_t launch_distance_maps(const float* pts, const long long* off, int K, int nx, int ny,
                                 int nz, const double sp[3], float* dmap, cudaStream_t s) {
  if (K == 0) return cudaSuccess;
  const long long V = (long long)nx * ny * nz;
  dim3 grid((unsigned)((V + 255) / 256), (unsigned)K);
  k_distance_maps<<<grid, 256, 0, s>>>(pts, off, K, nx, ny, nz, sp[0], sp[1], sp[2], dmap);
  return cudaGetLastError();
}

__global__ void k_band_mask(const float* __restrict__ dmap, int K, long long V, double r,
                            unsigned char* __restrict__ band) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < V;
       v += (long long)gridDim.x * blockDim.x) {
    unsigned m = 0;
    for (int i = 0; i < K; i++)
      if ((double)dmap[(long long)i * V + v] < r) m |= 1u << i;
    band[v] = (unsigned char)m;
  }
}

// own-side record per voxel: (bits of I(q), band bits) -> one 8-byte load per sample
__global__ void k_own_records(const float* __restrict__ I, const unsigned char* __restrict__ band, long long V,
                              uint2* __restrict__ out) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < V;
       v += (long long)gridDim.x * blockDim.x)
    out[v] = make_uint2(__float_as_uint(I[v]), band ? (unsigned)band[v] : 0u);
}

// zero radius of a volume by dilation: m = [I != 0], then per radius r = 1..15
// m = max over the 3x3x3 neighbourhood (one axis at a time), zr = the first r with m
__global__ void k_zr_init(const float* __restrict__ I, long long V, unsigned char* __restrict__ m,
                          unsigned char* __restrict__ zr) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < V;
       v += (long long)gridDim.x * blockDim.x) {
    const bool nz = I[v] != 0.0f;
    m[v] = nz ? 1 : 0;
    zr[v] = nz ? 0 : 15;
  }
}

__global__ void k_zr_dilate(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst, int nx,
                            int ny, int nz, int axis) {
  const long long V = (long long)nx * ny * nz;
  const long long st = axis == 0 ? 1 : (axis == 1 ? nx : (long long)nx * ny);
  const int n = axis == 0 ? nx : (axis == 1 ? ny : nz);
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < V;
       v += (long long)gridDim.x * blockDim.x) {
    const int c = axis == 0 ? (int)(v % nx) : (axis == 1 ? (int)((v / nx) % ny) : (int)(v / ((long long)nx * ny)));
    unsigned char x = src[v];
    if (c > 0) x |= src[v - st];
    if (c < n - 1) x |= src[v + st];
    dst[v] = x;
  }
}

__global__ void k_zr_update(const unsigned char* __restrict__ m, long long V, int r, unsigned char* __restrict__ zr) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < V;
       v += (long long)gridDim.x * blockDim.x)
    if (m[v] && zr[v] > r) zr[v] = (unsigned char)r;
}

// Row hulls of the non-quiet voxels of one side.  The quiet radius of voxel q is 0
// unless I(q) = 0 and q has no band entry, else zr(q) = the zero radius of the other
// volume (Chebyshev distance from q to its nearest non-zero voxel, boxes clipped to
// the image, 15 = at least 15).  Per image row (y, z) and radius R, the first and last
// x with quiet radius < R, (nx, -1) when there is none: a row interval outside that
// hull is quiet at R.  One thread per (row, R).
__global__ void k_quiet_hull(const float* __restrict__ I, const unsigned char* __restrict__ band,
                             const unsigned char* __restrict__ zr, int nx, int ny, int nz, short2* __restrict__ hull) {
  const int rows = ny * nz;
  const int nR = kQuietRmax - kQuietRmin + 1;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < rows * nR; t += gridDim.x * blockDim.x) {
    const int row = t % rows, R = kQuietRmin + t / rows;
    const long long base = (long long)row * nx;
    int first = nx, last = -1;
    for (int x = 0; x < nx; x++) {
      const long long v = base + x;
      const int q = (I[v] != 0.0f || (band && band[v])) ? 0 : zr[v];
      if (q < R) {
        first = min(first, x);
        last = x;
      }
    }
    hull[t] = make_short2((short)first, (short)last);
  }
}

// Per-voxel quiet radius q (as k_quiet_hull), then its minimum over the 4^3 block
// v - 1 .. v + 2 (clipped to the image), one axis at a time.
__global__ void k_quiet_voxel(const float* __restrict__ I, const unsigned char* __restrict__ band,
                              const unsigned char* __restrict__ zr, long long V, unsigned char* __restrict__ q) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < V;
       v += (long long)gridDim.x * blockDim.x)
    q[v] = (I[v] != 0.0f || (band && band[v])) ? 0 : zr[v];
}

__global__ void k_min4(const unsigned char* __restrict__ in, unsigned char* __restrict__ out, int n, long long stride,
                       long long V) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < V;
       v += (long long)gridDim.x * blockDim.x) {
    const int c = (int)((v / stride) % n);
    unsigned char m = in[v];
    if (c > 0) m = min(m, in[v - stride]);
    if (c + 1 < n) m = min(m, in[v + stride]);
    if (c + 2 < n) m = min(m, in[v + 2 * stride]);
    out[v] = m;
  }
}

cudaError_t launch_quiet_cells(const float* I, const unsigned char* band, const unsigned char* zr, int nx, int ny,
                               int nz, unsigned char* tmp0, unsigned char* tmp1, unsigned char* qcell, cudaStream_t s) {
  const long long V = (long long)nx * ny * nz;
  k_quiet_voxel<<<2048, 256, 0, s>>>(I, band, zr, V, tmp0);
  k_min4<<<2048, 256, 0, s>>>(tmp0, tmp1, nx, 1, V);
  k_min4<<<2048, 256, 0, s>>>(tmp1, tmp0, ny, nx, V);
  k_min4<<<2048, 256, 0, s>>>(tmp0, qcell, nz, (long long)nx * ny, V);
  return cudaGetLastError();
}

cudaError_t launch_quiet_hull(const float* I, const unsigned char* band, const unsigned char* zr, int nx, int ny,
                              int nz, short2* hull, cudaStream_t s) {
  const int n = ny * nz * (kQuietRmax - kQuietRmin + 1);
  k_quiet_hull<<<(n + 255) / 256, 256, 0, s>>>(I, band, zr, nx, ny, nz, hull);
  return cudaGetLastError();
}

cudaError_t launch_zero_radius(const float* I, int nx, int ny, int nz, unsigned char* zr, unsigned char* m0,
                               unsigned char* m1, cudaStream_t s) {
  const long long V = (long long)nx * ny * nz;
  k_zr_init<<<2048, 256, 0, s>>>(I, V, m0, zr);
  for (int r = 1; r < 15; r++) {
    k_zr_dilate<<<2048, 256, 0, s>>>(m0, m1, nx, ny, nz, 0);
    k_zr_dilate<<<2048, 256, 0, s>>>(m1, m0, nx, ny, nz, 1);
    k_zr_dilate<<<2048, 256, 0, s>>>(m0, m1, nx, ny, nz, 2);
    k_zr_update<<<2048, 256, 0, s>>>(m1, V, r, zr);
    unsigned char* t = m0; m0 = m1; m1 = t;
  }
  return cudaGetLastError();
}

// edge-padded copy of one volume for the gather textures (Volumes::texI):
// dst (nx+2p) x (ny+2p) x (nz+2p), dst(x+p, y+p, z+p) = src(clamp(x), clamp(y), clamp(z))
__global__ void k_pad_volume(const float* __restrict__ src, int nx, int ny, int nz, int pad,
                             float* __restrict__ dst) {
  const long long wp = nx + 2 * pad, hp = ny + 2 * pad, n = wp * hp * (long long)(nz + 2 * pad);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(t % wp) - pad, y = (int)((t / wp) % hp) - pad, z = (int)(t / (wp * hp)) - pad;
    const int cx = min(max(x, 0), nx - 1), cy = min(max(y, 0), ny - 1), cz = min(max(z, 0), nz - 1);
    dst[t] = src[((long long)cz * ny + cy) * nx + cx];
  }
}

cudaError_t launch_pad_volume(const float* src, int nx, int ny, int nz, int pad, float* dst, cudaStream_t s) {
  k_pad_volume<<<1184, 256, 0, s>>>(src, nx, ny, nz, pad, dst);
  return cudaGetLastError();
}

cudaError_t launch_own_records(const float* I, const unsigned char* band, long long V,
                               uint2* out, cudaStream_t s) {
  k_own_records<<<2048, 256, 0, s>>>(I, band, V, out);
  return cudaGetLastError();
}

cudaError_t launch_band_mask(const float* dmap, int K, long long V, double r, unsigned char* band,
                             cudaStream_t s) {
  k_band_mask<<<2048, 256, 0, s>>>(dmap, K, V, r, band);
  return cudaGetLastError();
}

#include "morea_repair.cuh"
#include "morea_export.cuh"
#include "morea_mix.cuh"

}  // namespace morea

#include "morea_sobol.cuh"

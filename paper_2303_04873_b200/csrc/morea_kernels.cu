// morea_kernels.cu -- sm_100a kernels of the MOREA hot path (arXiv 2303.04873).
//
// Rows of SURVEY.md §8(a) and where they live:
//   a0 load-time maps          k_distance_maps, k_band_mask, k_validate_volume
//   a1 genotype decode          canon_q (fp64, exact Q.10 rounding)
//   a2 per-tet geometry + fold  tet_setup / setup_side, k_check_folds
//   a3 magnitude                magnitude()
//   a4 ownership rasterizer     row_interval() + raster() (exact int64 intervals)
//   a5 map + sample + h         EvalSample (fp32 map, exact case split)
//   a6 guidance term            EvalSample (band mask + trilinear of the other map)
//   a7 reductions               warp shuffles (fixed order), k_reduce
//   a8 partial evaluation       k_eval in partial mode + k_reduce with base_acc
//   a9 fold check               k_check_folds
// The readings of the paper (O1..O13) are cited per function.
//
// Work decomposition: one warp evaluates one (solution, tet)
// item at a time, both sides; warps pull items from a global queue in
// solution-minor order (consecutive items = same tet, next solution) so the
// gathered bricks stay L1/L2-resident; tets are scheduled largest first.
// Inside an item the 32 lanes compute the exact x-intervals of 32 bbox rows,
// prefix-sum their lengths and then sweep the flattened samples 32 at a time,
// so lanes stay busy whatever the row lengths.
#include <cuda_runtime.h>

#include <cstdint>

#include "morea.h"
#include "morea_internal.h"

namespace morea {

typedef long long i64;
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

struct SideGeom {
  i64 nrm[4][3];   // inward normal of the face opposite vertex k (|n| < 2^41)
  int f0[4][3];    // a vertex of that face (Q units)
  int U[4][3];     // Q_other - Q_own per vertex
  i64 absdet;      // |Delta| (Q units^3)
  int lo[3], hi[3];  // lattice bbox clipped to the image
  double A[3][3];  // displacement gradient du_a/dq_b
  double d0[3];    // displacement at lo
  float eps[3];    // fp32 filter bound per axis (0 = exact translation axis)
  int ok;
};

struct WarpSmem {
  SideGeom G;
  int4 row_i[32];   // (exclusive prefix, linear index of row start, xl, y | z << 16)
  float4 row_d[32]; // displacement (fp32) at the row start
};

// ---------------------------------------------------------------------------
// a2: per-tet geometry of one side (O2, O3, O4).  Exact integer arithmetic:
// |Q| < 2^19.6 so edge components < 2^20, normals < 2^41, |Delta| < 2^62.6.
// ---------------------------------------------------------------------------
__device__ __forceinline__ i64 det3(const int Q[4][3]) {
  i64 a0 = Q[1][0] - Q[0][0], a1 = Q[1][1] - Q[0][1], a2 = Q[1][2] - Q[0][2];
  i64 b0 = Q[2][0] - Q[0][0], b1 = Q[2][1] - Q[0][1], b2 = Q[2][2] - Q[0][2];
  i64 c0 = Q[3][0] - Q[0][0], c1 = Q[3][1] - Q[0][1], c2 = Q[3][2] - Q[0][2];
  return a0 * (b1 * c2 - b2 * c1) - a1 * (b0 * c2 - b2 * c0) + a2 * (b0 * c1 - b1 * c0);
}

__device__ __forceinline__ int floordiv1024(int v) { return v >> 10; }          // arithmetic shift = floor
__device__ __forceinline__ int ceildiv1024(int v) { return -((-v) >> 10); }

__device__ void setup_side(const int Q[4][3], const int Qo[4][3], int nx, int ny, int nz,
                           SideGeom& G) {
  i64 det = det3(Q);
  G.ok = 0;
  if (det == 0) return;  // degenerate: owns nothing (O3)
  G.absdet = det < 0 ? -det : det;
  const int dims[3] = {nx, ny, nz};
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int f0 = (k == 0) ? 1 : 0;
    const int f1 = (k <= 1) ? 2 : 1;
    const int f2 = (k <= 2) ? 3 : 2;
    i64 u0 = Q[f1][0] - Q[f0][0], u1 = Q[f1][1] - Q[f0][1], u2 = Q[f1][2] - Q[f0][2];
    i64 v0 = Q[f2][0] - Q[f0][0], v1 = Q[f2][1] - Q[f0][1], v2 = Q[f2][2] - Q[f0][2];
    i64 n0 = u1 * v2 - u2 * v1, n1 = u2 * v0 - u0 * v2, n2 = u0 * v1 - u1 * v0;
    i64 s = n0 * (Q[k][0] - Q[f0][0]) + n1 * (Q[k][1] - Q[f0][1]) + n2 * (Q[k][2] - Q[f0][2]);
    if (s < 0) { n0 = -n0; n1 = -n1; n2 = -n2; }
    G.nrm[k][0] = n0; G.nrm[k][1] = n1; G.nrm[k][2] = n2;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      G.f0[k][a] = Q[f0][a];
      G.U[k][a] = Qo[k][a] - Q[k][a];
    }
  }
#pragma unroll
  for (int a = 0; a < 3; a++) {
    int mn = min(min(Q[0][a], Q[1][a]), min(Q[2][a], Q[3][a]));
    int mx = max(max(Q[0][a], Q[1][a]), max(Q[2][a], Q[3][a]));
    G.lo[a] = max(ceildiv1024(mn), 0);
    G.hi[a] = min(floordiv1024(mx), dims[a] - 1);
    if (G.lo[a] > G.hi[a]) return;
  }
  // O4: displacement u(p) = sum_k lambda_k(p) U_k / 1024, lambda_k = e_k / |Delta|,
  // e_k(p) = n_k . (1024 p - f0_k).  Gradient du_a/dp_b = sum_k n_kb U_ka / |Delta|.
  const double inv_det = 1.0 / (double)G.absdet;
  i64 elo[4];
#pragma unroll
  for (int k = 0; k < 4; k++) {
    elo[k] = G.nrm[k][0] * (i64)(1024 * G.lo[0] - G.f0[k][0]) +
             G.nrm[k][1] * (i64)(1024 * G.lo[1] - G.f0[k][1]) +
             G.nrm[k][2] * (i64)(1024 * G.lo[2] - G.f0[k][2]);
  }
#pragma unroll
  for (int a = 0; a < 3; a++) {
    bool exact = true;
#pragma unroll
    for (int b = 0; b < 3; b++) {
      i128 num = 0;
#pragma unroll
      for (int k = 0; k < 4; k++) num += (i128)G.nrm[k][b] * (i128)G.U[k][a];
      if (num != 0) exact = false;
      G.A[a][b] = (double)num * inv_det;
    }
    if (exact) {
      // every vertex moves by the same U_a: x_a = q_a + U_a / 1024 exactly
      G.d0[a] = (double)G.U[0][a] * (1.0 / 1024.0);
      G.eps[a] = 0.0f;
    } else {
      i128 N = 0;
#pragma unroll
      for (int k = 0; k < 4; k++) N += (i128)elo[k] * (i128)G.U[k][a];
      G.d0[a] = (double)N / (1024.0 * (double)G.absdet);
      // fp32 error bound of d = fma(A_x, k, d_row): 2^-24 (|d_row| + 2|A_x| k + |d|) + frac
      // rounding; Dmax bounds |u_a| over the bbox (affine => attained at a corner).
      double dmax = 0.0;
#pragma unroll
      for (int c = 0; c < 8; c++) {
        double v = G.d0[a] + G.A[a][0] * (double)((c & 1) ? G.hi[0] - G.lo[0] : 0) +
                   G.A[a][1] * (double)((c & 2) ? G.hi[1] - G.lo[1] : 0) +
                   G.A[a][2] * (double)((c & 4) ? G.hi[2] - G.lo[2] : 0);
        dmax = fmax(dmax, fabs(v));
      }
      double bound = dmax + fabs(G.A[a][0]) * (double)(G.hi[0] - G.lo[0]) + 1.0;
      G.eps[a] = (float)ldexp(bound, -22);  // 2x the bound, see DESIGN.md §4.3
    }
  }
  G.ok = 1;
}

// ---------------------------------------------------------------------------
// a4: exact x-interval of owned lattice points on row (y, z) (O3).  Face k owns
// the point iff e_k > 0, or e_k = 0 and lexpos(n_k) (perturbation q + (e,e^2,e^3)).
// Along x, e_k(x) = E0 + 1024 n_kx x; each face gives a half-line, found from an
// fp64 estimate and corrected by exact int64 evaluation.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void row_interval(const SideGeom& G, int y, int z, int& xl, int& xh) {
  const int lo = G.lo[0], hi = G.hi[0];
  xl = lo;
  xh = hi;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const i64 n0 = G.nrm[k][0], n1 = G.nrm[k][1], n2 = G.nrm[k][2];
    const i64 E0 = n1 * (i64)(1024 * y - G.f0[k][1]) + n2 * (i64)(1024 * z - G.f0[k][2]) -
                   n0 * (i64)G.f0[k][0];
    if (n0 > 0) {  // increasing; lexpos true: smallest x with e >= 0
      const i64 D = 1024 * n0;
      double est = ceil(-(double)E0 / (double)D);
      est = fmin(fmax(est, (double)lo), (double)(hi + 1));
      i64 x = (i64)est;
      while (x > lo && E0 + D * (x - 1) >= 0) --x;
      while (x <= hi && E0 + D * x < 0) ++x;
      xl = max(xl, (int)x);
    } else if (n0 < 0) {  // decreasing; lexpos false: largest x with e > 0
      const i64 D = 1024 * n0;
      double est = ceil((double)E0 / (double)(-D)) - 1.0;
      est = fmin(fmax(est, (double)(lo - 1)), (double)hi);
      i64 x = (i64)est;
      while (x < hi && E0 + D * (x + 1) > 0) ++x;
      while (x >= lo && E0 + D * x <= 0) --x;
      xh = min(xh, (int)x);
    } else {
      const bool own = E0 > 0 || (E0 == 0 && (n1 > 0 || (n1 == 0 && n2 > 0)));
      if (!own) xl = hi + 1;
    }
  }
}

// Generic rasterizer: calls f(row_info, row_disp, k) for every owned sample of
// the side, 32 samples per warp step.  All lanes of the warp must call it.
template <class F>
__device__ __forceinline__ void raster(const SideGeom& G, int nx, int ny, WarpSmem& S, int lane,
                                       F& f) {
  const int nyb = G.hi[1] - G.lo[1] + 1, nzb = G.hi[2] - G.lo[2] + 1;
  const int nrows = nyb * nzb;
  for (int r0 = 0; r0 < nrows; r0 += 32) {
    const int r = r0 + lane;
    int len = 0, xl = 0, y = 0, z = 0;
    float4 drow = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < nrows) {
      y = G.lo[1] + r % nyb;
      z = G.lo[2] + r / nyb;
      int xh;
      row_interval(G, y, z, xl, xh);
      len = max(0, xh - xl + 1);
      if (len) {
        const double ox = (double)(xl - G.lo[0]), oy = (double)(y - G.lo[1]),
                     oz = (double)(z - G.lo[2]);
        drow.x = (float)(G.d0[0] + G.A[0][0] * ox + G.A[0][1] * oy + G.A[0][2] * oz);
        drow.y = (float)(G.d0[1] + G.A[1][0] * ox + G.A[1][1] * oy + G.A[1][2] * oz);
        drow.z = (float)(G.d0[2] + G.A[2][0] * ox + G.A[2][1] * oy + G.A[2][2] * oz);
      }
    }
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(FULLMASK, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(FULLMASK, incl, 31);
    if (total == 0) continue;
    __syncwarp();
    S.row_i[lane] = make_int4(incl - len, (z * ny + y) * nx + xl, xl, y | (z << 16));
    S.row_d[lane] = drow;
    __syncwarp();
    for (int s0 = 0; s0 < total; s0 += 32) {
      const int idx = s0 + lane;
      int pos = 0;
#pragma unroll
      for (int b = 16; b; b >>= 1) {
        int v = __shfl_sync(FULLMASK, incl, pos + b - 1);
        if (v <= idx) pos += b;
      }
      if (idx < total) {
        const int4 ri = S.row_i[pos];
        const float4 rd = S.row_d[pos];
        f(ri, rd, idx - ri.x);
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// O6 slow path: exact contributing corner set when the fp32 position is within
// eps of a lattice plane on some axis.  x_a = (q_a M + N_a) / M exactly, with
// M = 1024 |Delta| and N_a = sum_k e_k(q) U_ka (int128).
// ---------------------------------------------------------------------------
__device__ __noinline__ bool exact_fg(const SideGeom& G, int qx, int qy, int qz, float dx, float dy,
                                      float dz, const float* __restrict__ vol, int nx, int ny,
                                      int nz) {
  const int q[3] = {qx, qy, qz};
  const float d[3] = {dx, dy, dz};
  const int dims[3] = {nx, ny, nz};
  i64 e[4];
  for (int k = 0; k < 4; k++)
    e[k] = G.nrm[k][0] * (i64)(1024 * qx - G.f0[k][0]) + G.nrm[k][1] * (i64)(1024 * qy - G.f0[k][1]) +
           G.nrm[k][2] * (i64)(1024 * qz - G.f0[k][2]);
  const i128 M = (i128)1024 * (i128)G.absdet;
  int cnt[3], idx[3][2];
  for (int a = 0; a < 3; a++) {
    i128 N = 0;
    for (int k = 0; k < 4; k++) N += (i128)e[k] * (i128)G.U[k][a];
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

// Per-axis clamp of the fp32 position (O5): returns i0 in [0, n-2] and weight
// f in [0, 1]; x <= 0 -> (0, 0) ; x >= n-1 -> (n-2, 1); otherwise floor / frac.
__device__ __forceinline__ void axis_clamp(int q, float d, int n, float eps, int& i0, float& f,
                                           bool& amb) {
  const float fl = floorf(d);
  float fr = d - fl;
  amb = (fr < eps) || (fr > 1.0f - eps);
  amb = amb && (eps > 0.0f);
  const int ix = q + (int)fl;
  if (ix < 0 || (ix == 0 && fr == 0.0f)) {
    i0 = 0; fr = 0.0f;
  } else if (ix >= n - 1) {
    i0 = n - 2; fr = 1.0f;
  } else {
    i0 = ix;
  }
  f = fr;
}

__device__ __forceinline__ float lerpf(float a, float b, float t) { return fmaf(t, b - a, a); }

// a5 + a6: one sample of one side.
struct EvalSample {
  const SideGeom& G;
  const float* __restrict__ Iown;
  const float* __restrict__ Ioth;
  const unsigned char* __restrict__ band;
  const float* __restrict__ dmap_own;
  const float* __restrict__ dmap_oth;
  long long V;
  int nx, ny, nz;
  float ax, ay, az;  // displacement gradient along x (fp32)
  float ex, ey, ez;  // per-axis filter bounds
  double r, inv_r;
  const double* w;   // pair weights of this side
  double h_sum, g_sum;
  int n, nb;

  __device__ __forceinline__ void operator()(const int4& ri, const float4& rd, int k) {
    const int qx = ri.z + k, qy = ri.w & 0xffff, qz = ri.w >> 16;
    const int lin = ri.y + k;
    const float a = __ldg(&Iown[lin]);
    const float dx = fmaf(ax, (float)k, rd.x);
    const float dy = fmaf(ay, (float)k, rd.y);
    const float dz = fmaf(az, (float)k, rd.z);
    int i0x, i0y, i0z;
    float fx, fy, fz;
    bool bx, by, bz;
    axis_clamp(qx, dx, nx, ex, i0x, fx, bx);
    axis_clamp(qy, dy, ny, ey, i0y, fy, by);
    axis_clamp(qz, dz, nz, ez, i0z, fz, bz);
    const long long sy = nx, sz = (long long)nx * ny;
    const long long base = i0z * sz + i0y * sy + i0x;
    const float c000 = __ldg(&Ioth[base]), c100 = __ldg(&Ioth[base + 1]);
    const float c010 = __ldg(&Ioth[base + sy]), c110 = __ldg(&Ioth[base + sy + 1]);
    const float c001 = __ldg(&Ioth[base + sz]), c101 = __ldg(&Ioth[base + sz + 1]);
    const float c011 = __ldg(&Ioth[base + sz + sy]), c111 = __ldg(&Ioth[base + sz + sy + 1]);
    const float b = lerpf(lerpf(lerpf(c000, c100, fx), lerpf(c010, c110, fx), fy),
                          lerpf(lerpf(c001, c101, fx), lerpf(c011, c111, fx), fy), fz);
    bool fg;
    if (bx || by || bz) {
      fg = exact_fg(G, qx, qy, qz, dx, dy, dz, Ioth, nx, ny, nz);
    } else {
      // contributing corners: lower corner iff f < 1, upper corner iff f > 0 (per axis)
      const unsigned m = (c000 > 0.f) | ((c100 > 0.f) << 1) | ((c010 > 0.f) << 2) |
                         ((c110 > 0.f) << 3) | ((c001 > 0.f) << 4) | ((c101 > 0.f) << 5) |
                         ((c011 > 0.f) << 6) | ((c111 > 0.f) << 7);
      const unsigned mx = (fx < 1.f ? 0x55u : 0u) | (fx > 0.f ? 0xAAu : 0u);
      const unsigned my = (fy < 1.f ? 0x33u : 0u) | (fy > 0.f ? 0xCCu : 0u);
      const unsigned mz = (fz < 1.f ? 0x0Fu : 0u) | (fz > 0.f ? 0xF0u : 0u);
      fg = (m & mx & my & mz) != 0u;
    }
    // h of PAPER.md §4.1.2 (L318-322) with the exact case split (O6)
    float h;
    if (a > 0.f && fg) {
      const float t = a - b;
      h = t * t;
    } else if (a == 0.f && !fg) {
      h = 0.f;
    } else {
      h = 1.f;
    }
    h_sum += (double)h;
    n += 1;
    if (band) {
      unsigned bm = __ldg(&band[lin]);
      nb += __popc(bm);
      while (bm) {
        const int i = __ffs(bm) - 1;
        bm &= bm - 1;
        const float* Do = dmap_oth + (long long)i * V;
        const float d = __ldg(&dmap_own[(long long)i * V + lin]);
        const float e000 = __ldg(&Do[base]), e100 = __ldg(&Do[base + 1]);
        const float e010 = __ldg(&Do[base + sy]), e110 = __ldg(&Do[base + sy + 1]);
        const float e001 = __ldg(&Do[base + sz]), e101 = __ldg(&Do[base + sz + 1]);
        const float e011 = __ldg(&Do[base + sz + sy]), e111 = __ldg(&Do[base + sz + sy + 1]);
        const float Dp = lerpf(lerpf(lerpf(e000, e100, fx), lerpf(e010, e110, fx), fy),
                               lerpf(lerpf(e001, e101, fx), lerpf(e011, e111, fx), fy), fz);
        const double dd = (double)d - (double)Dp;
        // O8: w_i (r - d)/r (d - D'(x))^2, only where d < r (band bit)
        g_sum += __ldg(&w[i]) * ((r - (double)d) * inv_r) * dd * dd;
      }
    }
  }
};

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

struct TetRes {
  double h, g, m, sev;
  long long n;
  int folds, flags, nb;
};

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
    const float* o = sl[k] >= 0 ? A.new_vals + ((long long)sol * A.S_total + sl[k]) * 6
                                : A.offsets + ((long long)sol * A.mesh.N + j) * 6;
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const float b = __ldg(&A.mesh.base[3 * j + a]);
#pragma unroll
      for (int s = 0; s < 2; s++) {
        const i64 q = canon_q(b, __ldg(&o[3 * s + a]));
        ok = ok && (q >= kQLo) && (q < kQHi);
        Q[s][k][a] = (int)q;
      }
    }
  }
  return ok;
}

// Evaluate one (solution, tet) item on the whole warp.  With raster = false
// only the per-tet terms (magnitude, folds) are computed.
__device__ TetRes eval_tet(const EvalArgs& A, WarpSmem& S, int lane, int sol, int tet, int4 slots,
                           bool do_raster) {
  TetRes R;
  R.h = R.g = R.m = R.sev = 0.0;
  R.n = 0;
  R.folds = R.flags = R.nb = 0;
  int Q[2][4][3];
  if (!load_tet(A, sol, A.mesh.tets[tet], slots, Q)) {
    R.flags = 1;
    return R;
  }
  const Volumes& V = A.vol;
  const double sp2[3] = {V.sp[0] * V.sp[0], V.sp[1] * V.sp[1], V.sp[2] * V.sp[2]};
  R.m = magnitude(Q, (double)__ldg(&A.mesh.cdelta[tet]), sp2, A.mesh.spoke_mode);
  const int ref = A.mesh.ref[tet];
  double h_sum = 0.0, g_sum = 0.0;
  int n = 0, nb = 0;
#pragma unroll 1
  for (int s = 0; s < 2; s++) {
    const i64 det = det3(Q[s]);
    const int sg = (det > 0) - (det < 0);
    if (sg != ref) {  // O2: sign change; zero counts as a fold
      R.folds += 1;
      const double vol = (double)(det < 0 ? -det : det) / (6.0 * 1073741824.0);
      R.sev += vol * V.sp[0] * V.sp[1] * V.sp[2];
    }
    if (!do_raster) continue;
    __syncwarp();
    if (lane == 0) setup_side(Q[s], Q[1 - s], V.nx, V.ny, V.nz, S.G);
    __syncwarp();
    if (!S.G.ok) continue;
    EvalSample f{S.G, V.I[s], V.I[1 - s], V.band[s], V.dmap[s], V.dmap[1 - s], V.V, V.nx, V.ny,
                 V.nz, (float)S.G.A[0][0], (float)S.G.A[1][0], (float)S.G.A[2][0], S.G.eps[0],
                 S.G.eps[1], S.G.eps[2], V.r, 1.0 / V.r, V.w + s * kMaxPairs, 0.0, 0.0, 0, 0};
    raster(S.G, V.nx, V.ny, S, lane, f);
    h_sum += f.h_sum;
    g_sum += f.g_sum;
    n += f.n;
    nb += f.nb;
  }
  if (do_raster) {
    R.h = warp_sum_d(h_sum);
    R.g = warp_sum_d(g_sum);
    R.n = warp_sum_i(n);
    R.nb = warp_sum_i(nb);
  }
  return R;
}

__global__ void __launch_bounds__(kEvalThreads) k_eval(const EvalArgs A) {
  __shared__ WarpSmem smem[kWarpsPerBlock];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmem& S = smem[warp];
  const long long n_items = (long long)A.n_entries * A.P;
  unsigned long long my_samples = 0, my_band = 0, my_items = 0;
  const int4 none = make_int4(-1, -1, -1, -1);
  while (true) {
    unsigned long long item = 0;
    if (lane == 0) item = atomicAdd(A.counter, 1ULL);
    item = __shfl_sync(FULLMASK, item, 0);
    if ((long long)item >= n_items) break;
    const int e = (int)(item / (unsigned long long)A.P);
    const int sol = (int)(item % (unsigned long long)A.P);
    const int tet = A.entry_tet[e];
    const int out = A.entry_out[e];
    Rec rec;
    if (!A.partial) {
      const TetRes R = eval_tet(A, S, lane, sol, tet, none, true);
      my_samples += R.n; my_band += R.nb; my_items += 1;
      rec.h = R.h; rec.g = R.g; rec.m = R.m; rec.sev = R.sev;
      rec.n = R.n; rec.folds = R.folds; rec.flags = R.flags;
      if (A.cache_out && lane < 4) {
        const double v = lane == 0 ? R.h : lane == 1 ? R.g : lane == 2 ? (double)R.n : R.m;
        A.cache_out[((long long)sol * A.mesh.T + tet) * 4 + lane] = v;
      }
    } else {
      const TetRes Rn = eval_tet(A, S, lane, sol, tet, A.entry_slots[e], true);
      TetRes Ro;
      if (A.cache_in) {
        Ro = eval_tet(A, S, lane, sol, tet, none, false);
        const double* c = A.cache_in + ((long long)sol * A.mesh.T + tet) * 4;
        Ro.h = c[0]; Ro.g = c[1]; Ro.n = (long long)c[2];
      } else {
        Ro = eval_tet(A, S, lane, sol, tet, none, true);
        my_samples += Ro.n; my_band += Ro.nb; my_items += 1;
      }
      my_samples += Rn.n; my_band += Rn.nb; my_items += 1;
      rec.h = Rn.h - Ro.h; rec.g = Rn.g - Ro.g; rec.m = Rn.m - Ro.m; rec.sev = Rn.sev - Ro.sev;
      rec.n = Rn.n - Ro.n; rec.folds = Rn.folds - Ro.folds; rec.flags = Rn.flags;
      if (A.cache_out && lane < 4) {
        const double v = lane == 0 ? Rn.h : lane == 1 ? Rn.g : lane == 2 ? (double)Rn.n : Rn.m;
        A.cache_out[((long long)sol * A.n_out + out) * 4 + lane] = v;
      }
    }
    if (lane == 0) A.rec[(long long)sol * A.n_out + out] = rec;
  }
  if (lane == 0 && A.stats) {
    atomicAdd(&A.stats[0], my_samples);
    atomicAdd(&A.stats[1], my_band);
    atomicAdd(&A.stats[2], my_items);
  }
}

int eval_blocks_per_sm() {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_eval, kEvalThreads, 0) != cudaSuccess)
    return 1;
  return nb > 0 ? nb : 1;
}

cudaError_t launch_eval(const EvalArgs& a, int grid, cudaStream_t s) {
  k_eval<<<grid, kEvalThreads, 0, s>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// a7 / a8: per (solution, group) reduction in a fixed order (warp per output),
// objectives and flags.
// ---------------------------------------------------------------------------
__global__ void k_reduce(int P, int G, int n_out, const int* __restrict__ group_off,
                         const Rec* __restrict__ rec, const morea_acc* __restrict__ base_acc,
                         int partial, int T, int N, const float* __restrict__ base,
                         const float* __restrict__ offsets, const int* __restrict__ changed,
                         const int* __restrict__ grp_off, const float* __restrict__ new_vals,
                         int S_total, double* __restrict__ obj, morea_acc* __restrict__ acc) {
  const int lane = threadIdx.x & 31;
  const long long wid = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (wid >= (long long)P * G) return;
  const int sol = (int)(wid / G), g = (int)(wid % G);
  double h = 0.0, gs = 0.0, m = 0.0, sev = 0.0;
  long long n = 0;
  int folds = 0, flags = 0;
  const Rec* r = rec + (long long)sol * n_out;
  for (int e = group_off[g] + lane; e < group_off[g + 1]; e += 32) {
    const Rec x = r[e];
    h += x.h; gs += x.g; m += x.m; sev += x.sev; n += x.n; folds += x.folds; flags |= x.flags;
  }
  // domain check of the points that define this output (all points for a full
  // evaluation, the new values of S_g for a partial one)
  int dom = flags & 1;
  if (!partial) {
    for (int j = lane; j < N; j += 32)
      for (int c = 0; c < 6; c++) {
        const i64 q = canon_q(base[3 * j + (c % 3)], offsets[((long long)sol * N + j) * 6 + c]);
        if (q < kQLo || q >= kQHi) dom = 1;
      }
  } else {
    for (int i = grp_off[g] + lane; i < grp_off[g + 1]; i += 32) {
      const int j = changed[i];
      for (int c = 0; c < 6; c++) {
        const i64 q = canon_q(base[3 * j + (c % 3)], new_vals[((long long)sol * S_total + i) * 6 + c]);
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
    folds += __shfl_xor_sync(FULLMASK, folds, o);
    dom |= __shfl_xor_sync(FULLMASK, dom, o);
  }
  if (lane != 0) return;
  morea_acc out;
  if (partial) {
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
  }
  if (out.n_samples == 0) out.flags |= MOREA_F_EMPTY;
  const long long o = (long long)sol * G + g;
  if (acc) acc[o] = out;
  if (obj) {
    if (out.flags & (MOREA_F_DOMAIN | MOREA_F_EMPTY)) {
      obj[3 * o] = obj[3 * o + 1] = obj[3 * o + 2] = __longlong_as_double(0x7ff8000000000000LL);
    } else {
      obj[3 * o + 0] = out.m_sum / (10.0 * (double)T);          // L258
      obj[3 * o + 1] = out.h_sum / (double)out.n_samples;       // L317
      obj[3 * o + 2] = out.g_sum / (double)out.n_samples;       // L339
    }
  }
}

cudaError_t launch_reduce(int P, int G, int n_out, const int* group_off, const Rec* rec,
                          const void* base_acc, int partial, int T, int N, const float* base,
                          const float* offsets, const int* changed, const int* grp_off,
                          const float* new_vals, int S_total, double* obj, void* acc,
                          cudaStream_t s) {
  const long long warps = (long long)P * G;
  const int threads = 256;
  const long long blocks = (warps * 32 + threads - 1) / threads;
  k_reduce<<<(unsigned)blocks, threads, 0, s>>>(P, G, n_out, group_off, rec,
                                                (const morea_acc*)base_acc, partial, T, N, base,
                                                offsets, changed, grp_off, new_vals, S_total, obj,
                                                (morea_acc*)acc);
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
    for (int k = 0; k < 4; k++)
      for (int a = 0; a < 3; a++)
        for (int s = 0; s < 2; s++) {
          const i64 q = canon_q(M.base[3 * vid[k] + a], offsets[((long long)sol * M.N + vid[k]) * 6 + 3 * s + a]);
          ok = ok && q >= kQLo && q < kQHi;
          Q[s][k][a] = (int)q;
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
// Owner-map test hook: the same setup + rasterizer, one warp per tet.
// ---------------------------------------------------------------------------
struct OwnerSample {
  int* owner;
  int tet;
  __device__ __forceinline__ void operator()(const int4& ri, const float4&, int k) {
    const int lin = ri.y + k;
    const int old = atomicCAS(&owner[lin], -1, tet);
    if (old != -1) atomicExch(&owner[lin], -2);
  }
};

__global__ void __launch_bounds__(kEvalThreads) k_owner_map(Volumes V, MeshDev M,
                                                            const float* __restrict__ off, int side,
                                                            int* __restrict__ owner) {
  __shared__ WarpSmem smem[kWarpsPerBlock];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tet = blockIdx.x * kWarpsPerBlock + warp;
  if (tet >= M.T) return;
  WarpSmem& S = smem[warp];
  EvalArgs A;
  A.mesh = M;
  A.offsets = off;
  A.new_vals = nullptr;
  A.S_total = 0;
  int Q[2][4][3];
  if (!load_tet(A, 0, M.tets[tet], make_int4(-1, -1, -1, -1), Q)) return;
  if (lane == 0) setup_side(Q[side], Q[1 - side], V.nx, V.ny, V.nz, S.G);
  __syncwarp();
  if (!S.G.ok) return;
  OwnerSample f{owner, tet};
  raster(S.G, V.nx, V.ny, S, lane, f);
}

__global__ void k_fill_int(int* p, long long n, int v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) p[i] = v;
}

cudaError_t launch_owner_map(const Volumes& v, const MeshDev& m, const float* offsets_one,
                             int side, int* owner, cudaStream_t s) {
  k_fill_int<<<1024, 256, 0, s>>>(owner, v.V, -1);
  const int blocks = (m.T + kWarpsPerBlock - 1) / kWarpsPerBlock;
  k_owner_map<<<blocks, kEvalThreads, 0, s>>>(v, m, offsets_one, side, owner);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// a0: load-time work.
// ---------------------------------------------------------------------------
__global__ void k_validate_volume(const float* __restrict__ I, long long V, int* bad) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < V;
       i += (long long)gridDim.x * blockDim.x) {
    const float v = I[i];
    if (!(v >= 0.0f) || isinf(v)) atomicOr(bad, 1);
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

cudaError_t launch_band_mask(const float* dmap, int K, long long V, double r, unsigned char* band,
                             cudaStream_t s) {
  k_band_mask<<<2048, 256, 0, s>>>(dmap, K, V, r, band);
  return cudaGetLastError();
}

}  // namespace morea

// morea_sweep.cuh -- rows a2 (per-lane geometry), a4 (exactly-once ownership), a5
// (map + trilinear + h), a6 (guidance) and the per-tet part of a7 for the
// voxel-centre sample set, on sm_100a.  Included by morea_kernels.cu (inside
// namespace morea).
//
// Work decomposition.  One warp per item = (version, canonical
// entry, z-slab, group of 32 consecutive solutions); lane l evaluates solution
// 32 g + l.  The solutions of a population are near one another, so the 32 lanes
// see nearly the same tet: the warp walks the UNION of their lattice rows
// (warp-uniform z, y, x loops) and lane l counts a voxel q only where q lies in
// its own exact x-interval.  Consequences:
//   * the own record (I_side(q), band bits) is one broadcast load per step, and
//     the band bits are warp-uniform, so the guidance entries of a step are
//     evaluated in place (no queue): each lane gathers the other side's map at
//     its own position;
//   * per sample a lane pays only the map, the two tld4 gathers, the trilinear
//     interpolation and h -- no row lookup, no prefix sums, no shared tables;
//   * each lane's row interval is exact (fp32 face crossings with a derived
//     error bound, int64 decision from the lane's Q.10 vertices when a crossing
//     is within the bound of an integer), so ownership is exactly the oracle's
//     (reading O3) for every lane, whatever the other lanes do.
// Large tets are split into z-slabs on the host so no single item dominates a
// launch (slab sums are added in a fixed order by k_reduce).
#pragma once

#ifndef MOREA_SWEEP_WARPS
#define MOREA_SWEEP_WARPS 20  // warps of the one k_sweep block per SM (96 registers: no spills in the sample loop)
#endif

constexpr int kSweepWarps = MOREA_SWEEP_WARPS;
constexpr int kSweepThreads = 32 * kSweepWarps;

// ---------------------------------------------------------------------------
// a2 exact face geometry of one side from its Q.10 vertices (O2, O3, O4).
// |Q| < 2^19.6 so edge components < 2^20, normals < 2^41, |Delta| < 2^62.6 and
// e_k(q) < 3 2^61 for lattice points q of the Q.10 window.  Face k is opposite
// vertex k; its normal points inward (towards vertex k).
// ---------------------------------------------------------------------------
struct ExactFaces {
  i64 nrm[4][3];
  i64 cst[4];  // e_k(q) = 1024 n_k . q - cst_k
};

__device__ __forceinline__ void exact_faces(const int Q[4][3], ExactFaces& F) {
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int f0 = (k == 0) ? 1 : 0;
    const int f1 = (k <= 1) ? 2 : 1;
    const int f2 = (k <= 2) ? 3 : 2;
    const i64 u0 = Q[f1][0] - Q[f0][0], u1 = Q[f1][1] - Q[f0][1], u2 = Q[f1][2] - Q[f0][2];
    const i64 v0 = Q[f2][0] - Q[f0][0], v1 = Q[f2][1] - Q[f0][1], v2 = Q[f2][2] - Q[f0][2];
    i64 n0 = u1 * v2 - u2 * v1, n1 = u2 * v0 - u0 * v2, n2 = u0 * v1 - u1 * v0;
    const i64 s = n0 * (Q[k][0] - Q[f0][0]) + n1 * (Q[k][1] - Q[f0][1]) + n2 * (Q[k][2] - Q[f0][2]);
    if (s < 0) { n0 = -n0; n1 = -n1; n2 = -n2; }
    F.nrm[k][0] = n0; F.nrm[k][1] = n1; F.nrm[k][2] = n2;
    F.cst[k] = n0 * (i64)Q[f0][0] + n1 * (i64)Q[f0][1] + n2 * (i64)Q[f0][2];
  }
}

__device__ __forceinline__ i64 face_eval(const ExactFaces& F, int k, int x, int y, int z) {
  return 1024 * (F.nrm[k][0] * x + F.nrm[k][1] * y + F.nrm[k][2] * z) - F.cst[k];
}

__device__ __forceinline__ void lane_q(const LaneQ& L, int side, int Q[4][3]) {
#pragma unroll
  for (int k = 0; k < 4; k++)
#pragma unroll
    for (int a = 0; a < 3; a++) Q[k][a] = L.q[side][k][a];
}

// ceil(a / b) for b > 0 (int64, exact)
__device__ __forceinline__ i64 ceil_div_pos(i64 a, i64 b) {
  i64 q = a / b;  // truncation: already the ceiling for a <= 0
  if (a > 0 && q * b != a) q += 1;
  return q;
}

// O3 exact x-interval of row (y, z): face k owns q iff e_k(q) > 0, or e_k(q) = 0
// and lexpos(n_k) (the perturbation q + (e, e^2, e^3)).  Along x, e_k = m x + C
// with m = 1024 n_kx: a half-line (m != 0) or a row-constant decision (m = 0).
// Clipped to [lo, hi].  (Rare path: irregular faces, or a fast crossing within
// its error bound of an integer.)
__device__ __noinline__ int2 row_exact(const LaneQ* LQ, int side, int y, int z, int lo, int hi) {
  int Q[4][3];
  lane_q(*LQ, side, Q);
  ExactFaces F;
  exact_faces(Q, F);
  i64 xl = lo, xh = hi;
  for (int k = 0; k < 4; k++) {
    const i64 C = face_eval(F, k, 0, y, z);
    const i64 n0 = F.nrm[k][0];
    if (n0 == 0) {
      const bool lex = F.nrm[k][1] > 0 || (F.nrm[k][1] == 0 && F.nrm[k][2] > 0);
      if (!(C > 0 || (C == 0 && lex))) xh = lo - 1;
    } else if (n0 > 0) {  // lexpos: e = m x + C >= 0  <=>  x >= ceil(-C / m)
      xl = max(xl, ceil_div_pos(-C, 1024 * n0));
    } else {              // e = -m x + C > 0  <=>  x < C / m  <=>  x <= ceil(C / m) - 1
      xh = min(xh, ceil_div_pos(C, -1024 * n0) - 1);
    }
  }
  if (xl > xh) return make_int2(1, 0);
  return make_int2((int)xl, (int)xh);
}

// all lanes call it (warp-uniform branch); lanes with ex = false keep r
__device__ __noinline__ int2 row_exact_if(bool ex, int2 r, const LaneQ* LQ, int side, int y, int z, int lo,
                                          int hi) {
  if (!ex) return r;
  return row_exact(LQ, side, y, z, lo, hi);
}

// O6 slow path: the exact contributing corner set of the clamped trilinear
// footprint at x = T(q) (x_a = (q_a M + N_a) / M exactly, M = 1024 |Delta|,
// N_a = sum_k e_k(q) U_ka in int128), then fg = some contributing corner > 0.
__device__ __forceinline__ bool exact_fg(const LaneQ* LQ, int side, int qx, int qy, int qz, float dx, float dy,
                                         float dz, const float* __restrict__ vol, int nx, int ny, int nz) {
  int Q[4][3], Qo[4][3];
  lane_q(*LQ, side, Q);
  lane_q(*LQ, 1 - side, Qo);
  ExactFaces F;
  exact_faces(Q, F);
  i64 det = det3(Q);
  if (det < 0) det = -det;
  const int q[3] = {qx, qy, qz};
  const float d[3] = {dx, dy, dz};
  const int dims[3] = {nx, ny, nz};
  i64 e[4];
  for (int k = 0; k < 4; k++) e[k] = face_eval(F, k, qx, qy, qz);
  const i128 M = (i128)1024 * (i128)det;
  int cnt[3], idx[3][2];
  for (int a = 0; a < 3; a++) {
    i128 N = 0;
    for (int k = 0; k < 4; k++) N += (i128)e[k] * (i128)(Qo[k][a] - Q[k][a]);
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

// (inlined under a warp-uniform branch: a call inside the sample loop would force
// the loop's live values into callee-saved registers or local memory)

// ---------------------------------------------------------------------------
// The fast fp32 view of one lane's tet side (built once per item and side).
// ---------------------------------------------------------------------------
struct LaneFast {
  float fa[4], fb[4], fc[4], thr[4];  // crossing x*(y,z) = fa + fb (y - lo_y) + fc (z - lo_z), bound thr
  float A[3][3];                      // displacement gradient du_a / dq_b
  float d0[3];                        // displacement at lo
  float eps[3];                       // position filter bound per axis (0 = exact axis)
  float vy[4], vz[4];                 // vertex y, z (exact) for the slice y ranges
  int lo[3], hi[3];                   // lattice bbox clipped to the image
  int flags;                          // bit 0: rasterize; 1: positions inside [0, n-1) (plain loads
                                      // need no clamp); 2: all faces regular (fast rows); 3: positions
                                      // inside (-1, n) (edge-padded textures need no clamp)
};

// a2 for one side (O3, O4): faces, fp32 crossings with error bounds, the
// displacement-form affine map with its fp32 error bound, clamp flags.
__device__ __noinline__ void build_lane(const int Q[4][3], const int Qo[4][3], int nx, int ny, int nz,
                                        LaneFast& G) {
  G.flags = 0;
#pragma unroll
  for (int a = 0; a < 3; a++) { G.lo[a] = 1; G.hi[a] = 0; }
  const i64 det = det3(Q);
  if (det == 0) return;  // degenerate: owns nothing (O3)
  const i64 absdet = det < 0 ? -det : det;
  const int dims[3] = {nx, ny, nz};
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const int mn = min(min(Q[0][a], Q[1][a]), min(Q[2][a], Q[3][a]));
    const int mx = max(max(Q[0][a], Q[1][a]), max(Q[2][a], Q[3][a]));
    G.lo[a] = max(ceildiv1024(mn), 0);
    G.hi[a] = min(floordiv1024(mx), dims[a] - 1);
  }
  if (G.lo[0] > G.hi[0] || G.lo[1] > G.hi[1] || G.lo[2] > G.hi[2]) return;  // no lattice point inside
  ExactFaces F;
  exact_faces(Q, F);
  const double Ly = (double)(G.hi[1] - G.lo[1]), Lz = (double)(G.hi[2] - G.lo[2]);
  bool regular = true;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    G.vy[k] = (float)Q[k][1] * (1.0f / 1024.0f);  // exact: |Q| < 2^20
    G.vz[k] = (float)Q[k][2] * (1.0f / 1024.0f);
    const i64 n0 = F.nrm[k][0], n1 = F.nrm[k][1], n2 = F.nrm[k][2];
    if (n0 != 0) {
      // row crossing x*(y, z): 1024 (n0 x + n1 y + n2 z) = cst
      const i128 num = (i128)F.cst[k] - (i128)1024 * ((i128)n1 * G.lo[1] + (i128)n2 * G.lo[2]);
      const double fa = (double)num / (1024.0 * (double)n0);
      const double fb = -(double)n1 / (double)n0, fc = -(double)n2 / (double)n0;
      G.fa[k] = (float)fa;
      G.fb[k] = (float)fb;
      G.fc[k] = (float)fc;
      // fp32 rounding of 3 coefficients + 2 fma: < 2^-22 (|fa| + |fb| Ly + |fc| Lz); 4x margin
      const double thr = ldexp(fabs(fa) + fabs(fb) * Ly + fabs(fc) * Lz + 1.0, -20);
      // the sign of the bound says which side the face bounds: + lower (n0 > 0), - upper
      G.thr[k] = n0 > 0 ? (float)thr : -(float)thr;
      regular = regular && thr < 0.25;
    } else {
      G.fa[k] = G.fb[k] = G.fc[k] = 0.f;
      G.thr[k] = 1.0f;
      regular = false;
    }
  }
  // O4: displacement u(p) = sum_k lambda_k U_k / 1024, lambda_k = e_k / |Delta|.
  // Gradient du_a/dp_b = sum_k n_kb U_ka / |Delta|; value at lo from exact e_k(lo).
  const double inv_det = 1.0 / (double)absdet;
  const double L[3] = {(double)(G.hi[0] - G.lo[0]), Ly, Lz};
  i64 elo[4];
#pragma unroll
  for (int k = 0; k < 4; k++) elo[k] = face_eval(F, k, G.lo[0], G.lo[1], G.lo[2]);
  bool inside = true;   // positions in [0, n-1) (plain loads need no clamp)
  bool inside_p = true; // positions in (-1, n) (edge-padded textures need no clamp)
#pragma unroll
  for (int a = 0; a < 3; a++) {
    bool exact = true;
    double Aab[3];
#pragma unroll
    for (int b = 0; b < 3; b++) {
      i128 num = 0;
#pragma unroll
      for (int k = 0; k < 4; k++) num += (i128)F.nrm[k][b] * (i128)(Qo[k][a] - Q[k][a]);
      if (num != 0) exact = false;
      Aab[b] = (double)num * inv_det;
      G.A[a][b] = (float)Aab[b];
    }
    if (exact) {
      // every vertex moves by the same U_a: x_a = q_a + U_a / 1024 exactly (fp32-exact)
      G.d0[a] = (float)(Qo[0][a] - Q[0][a]) * (1.0f / 1024.0f);
      G.eps[a] = 0.0f;
    } else {
      i128 N = 0;
#pragma unroll
      for (int k = 0; k < 4; k++) N += (i128)elo[k] * (i128)(Qo[k][a] - Q[k][a]);
      const double d0 = (double)N / (1024.0 * (double)absdet);
      G.d0[a] = (float)d0;
      double amax = 0.0;
#pragma unroll
      for (int c = 0; c < 8; c++) {
        const double v = d0 + Aab[0] * ((c & 1) ? L[0] : 0.0) + Aab[1] * ((c & 2) ? L[1] : 0.0) +
                         Aab[2] * ((c & 4) ? L[2] : 0.0);
        amax = fmax(amax, fabs(v));
      }
      // fp32 error of d = fma(A_x0, k, d_row) with d_row = fma(A_a0, ox, fma(A_a1, oy,
      // fma(A_a2, oz, d0))) and of frac(d): every partial sum is a displacement at a
      // bbox point (|.| <= amax); <= 2^-24 (5 (amax + sum_b |A_ab| L_b) + 1); eps = 3x
      const double bound = amax + fabs(Aab[0]) * L[0] + fabs(Aab[1]) * L[1] + fabs(Aab[2]) * L[2] + 1.0;
      G.eps[a] = (float)ldexp(bound, -19);
    }
    // An owned sample q lies in the closed tet, so x = T(q) lies in the other
    // side's vertex bbox; the margin covers the fp32 position error.
    const int omn = min(min(Qo[0][a], Qo[1][a]), min(Qo[2][a], Qo[3][a]));
    const int omx = max(max(Qo[0][a], Qo[1][a]), max(Qo[2][a], Qo[3][a]));
    const double xmin = (double)omn / 1024.0, xmax = (double)omx / 1024.0;
    const double mg = 1e-3 + 2.0 * (double)G.eps[a];
    if (!(xmin >= mg && xmax <= (double)(dims[a] - 1) - mg)) inside = false;
    if (!(xmin >= -1.0 + mg && xmax <= (double)dims[a] - mg)) inside_p = false;
  }
  G.flags = 1 | (inside ? 2 : 0) | (regular ? 4 : 0) | (inside_p ? 8 : 0);
}

// Conservative y range of the lane's tet cross-section with the plane z (exact
// vertex coordinates; edge intersections in fp32 with a 1e-3 voxel margin).
__device__ __forceinline__ void slice_y_range(const float4 vy, const float4 vz, int lo_y, int hi_y, int z,
                                              int& ylo, int& yhi) {
  const float Y[4] = {vy.x, vy.y, vy.z, vy.w};
  const float Z[4] = {vz.x, vz.y, vz.z, vz.w};
  float ymin = 3.0e38f, ymax = -3.0e38f;
  const float zf = (float)z;
#pragma unroll
  for (int i = 0; i < 4; i++) {
#pragma unroll
    for (int j = i + 1; j < 4; j++) {
      const float lo = fminf(Z[i], Z[j]), hi = fmaxf(Z[i], Z[j]);
      const bool in = zf >= lo && zf <= hi;
      float y0, y1;
      if (hi > lo) {
        const float t = __fdividef(zf - Z[i], Z[j] - Z[i]);  // ~2 ulp: covered by the 1e-3 margin
        y0 = y1 = fmaf(t, Y[j] - Y[i], Y[i]);
      } else {
        y0 = Y[i];
        y1 = Y[j];
      }
      ymin = in ? fminf(ymin, fminf(y0, y1)) : ymin;
      ymax = in ? fmaxf(ymax, fmaxf(y0, y1)) : ymax;
    }
  }
  ylo = max(lo_y, (int)ceilf(fmaxf(ymin - 1e-3f, -1.0e6f)));
  yhi = min(hi_y, (int)floorf(fminf(ymax + 1e-3f, 1.0e6f)));
}

__device__ __forceinline__ float lerp_p(float a, float b, float t, float omt) {
  // Positivity-exact lerp (1 - t) a + t b as fma(t, b, (1 - t) a): for a, b >= 0 and
  // t in [0, 1] it is > 0 iff a contributing value (a with t < 1, b with t > 0) is
  // > 0, barring underflow (excluded: non-zero intensities >= 2^-40).
  return fmaf(t, b, omt * a);
}

__device__ __forceinline__ float tri8(const float c[8], float fx, float fy, float fz, float gx, float gy,
                                      float gz) {
  return lerp_p(lerp_p(lerp_p(c[0], c[1], fx, gx), lerp_p(c[2], c[3], fx, gx), fy, gy),
                lerp_p(lerp_p(c[4], c[5], fx, gx), lerp_p(c[6], c[7], fx, gx), fy, gy), fz, gz);
}

__device__ __forceinline__ void gather2(unsigned long long tex, float u, float v, float fnyp, float c[8]) {
  const float4 g0 = tex2Dgather<float4>((cudaTextureObject_t)tex, u, v, 0);
  const float4 g1 = tex2Dgather<float4>((cudaTextureObject_t)tex, u, v + fnyp, 0);
  // gather order: (x0,y1) (x1,y1) (x1,y0) (x0,y0)
  c[0] = g0.w; c[1] = g0.z; c[2] = g0.x; c[3] = g0.y;
  c[4] = g1.w; c[5] = g1.z; c[6] = g1.x; c[7] = g1.y;
}

// Two samples' footprints (four tld4) issued back to back, so both samples' gathers
// are in flight together (the compiler otherwise consumes the first pair before
// issuing the second).
__device__ __forceinline__ void gather2x2(unsigned long long tex, float u0, float v0, float u1, float v1, float fnyp,
                                          float c0[8], float c1[8]) {
  float4 g0, g1, g2, g3;
  asm volatile(
      "tld4.r.2d.v4.f32.f32 {%0, %1, %2, %3}, [%16, {%17, %18}];\n\t"
      "tld4.r.2d.v4.f32.f32 {%4, %5, %6, %7}, [%16, {%17, %19}];\n\t"
      "tld4.r.2d.v4.f32.f32 {%8, %9, %10, %11}, [%16, {%20, %21}];\n\t"
      "tld4.r.2d.v4.f32.f32 {%12, %13, %14, %15}, [%16, {%20, %22}];"
      : "=f"(g0.x), "=f"(g0.y), "=f"(g0.z), "=f"(g0.w), "=f"(g1.x), "=f"(g1.y), "=f"(g1.z), "=f"(g1.w),
        "=f"(g2.x), "=f"(g2.y), "=f"(g2.z), "=f"(g2.w), "=f"(g3.x), "=f"(g3.y), "=f"(g3.z), "=f"(g3.w)
      : "l"(tex), "f"(u0), "f"(v0), "f"(v0 + fnyp), "f"(u1), "f"(v1), "f"(v1 + fnyp));
  // gather order: (x0,y1) (x1,y1) (x1,y0) (x0,y0)
  c0[0] = g0.w; c0[1] = g0.z; c0[2] = g0.x; c0[3] = g0.y;
  c0[4] = g1.w; c0[5] = g1.z; c0[6] = g1.x; c0[7] = g1.y;
  c1[0] = g2.w; c1[1] = g2.z; c1[2] = g2.x; c1[3] = g2.y;
  c1[4] = g3.w; c1[5] = g3.z; c1[6] = g3.x; c1[7] = g3.y;
}

__device__ __forceinline__ void load8(const float* __restrict__ vol, int base, int sy, int sz, float c[8]) {
  c[0] = __ldg(&vol[base]); c[1] = __ldg(&vol[base + 1]);
  c[2] = __ldg(&vol[base + sy]); c[3] = __ldg(&vol[base + sy + 1]);
  c[4] = __ldg(&vol[base + sz]); c[5] = __ldg(&vol[base + sz + 1]);
  c[6] = __ldg(&vol[base + sz + sy]); c[7] = __ldg(&vol[base + sz + sy + 1]);
}

// ---------------------------------------------------------------------------
// Per-lane state of the sweep.  Only what a sample needs stays in registers
// (SampleK and the row's RowCtx); the per-row and per-slice fields of the lanes
// live in the warp's shared memory (SoA [field][lane], read back per row with
// volatile loads so they are not kept live across the sample loop), the fp64
// sums too.
// ---------------------------------------------------------------------------
struct SampleK {
  float A00, A10, A20;  // du / dx
  float t0, t1, t2;     // 0.5 - eps per axis (ambiguity thresholds on |frac - 0.5|)
};

struct WarpLanes {
  float4 fb[32], thr[32];  // per row: face slopes fb_k, signed bounds thr_k (+ lower, - upper)
  float4 k1[32];           // (A01, A11, A21, bits (lo_x | hi_x << 10 | lo_y << 20))
  float4 zb[32];           // per slice: face crossings at (lo_y, z)
  float4 zt[32];           // per slice: (displacement at (lo_x, lo_y, z), bits (ylo | yhi << 16))
  double2 acc[32];         // (sum h, sum g) of the current item
  int2 cnt[32];            // (samples, side-0 samples) of the current item
  unsigned long long nb, steps;  // band entries, warp-steps (profiling)
};
static_assert(sizeof(WarpLanes) == 3344, "WarpLanes layout");

__device__ __forceinline__ float4 lds4(const float4* p) {
  float4 v;
  const unsigned a = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

// Row data handed to the row functors.
struct RowCtx {
  int side, z, y, X0, X1;  // warp-uniform
  int xl, xh;              // the lane's exact interval (xl > xh: empty)
  float dx, dy, dz;        // the lane's displacement at (xl, y, z)
};

// One sample's position in the other volume (O4, O5): the fp32 displacement
// d = fma(A_x0, kf, d_row), its floor and fractional parts, the ambiguity test
// (some fractional part within eps of a lattice plane: O6 must be decided
// exactly) and the gather coordinates of the footprint's lower corner.  Shared
// by the main pass and the exact pass, so both see the same fp32 values.
struct SamplePos {
  float dx, dy, dz, fx, fy, fz, u, v;
  int base;
  bool amb;
};

// What the per-sample helpers read of the volumes (Volumes itself in the kernel,
// where its fields are kernel-parameter operands; this by-value copy in the
// out-of-line exact pass, so the kernel parameters are never address-taken).
struct VolLite {
  int nx, ny, nz;
  long long V;
  float fnx2, fny2, fnz2, fnyp, voff;
  float uoffI[2];
  unsigned long long texI;
  const float* I[2];
  const uint2* own0;
};

template <bool TEX, bool CLAMP, class VT>
__device__ __forceinline__ SamplePos sample_pos(const VT& V, const SampleK& K, const RowCtx& r, int x, float kf,
                                                float vrow, float uoff) {
  SamplePos p;
  p.dx = fmaf(K.A00, kf, r.dx);
  p.dy = fmaf(K.A10, kf, r.dy);
  p.dz = fmaf(K.A20, kf, r.dz);
  const float flx = floorf(p.dx), fly = floorf(p.dy), flz = floorf(p.dz);
  p.fx = p.dx - flx;
  p.fy = p.dy - fly;
  p.fz = p.dz - flz;
  p.amb = (fabsf(p.fx - 0.5f) > K.t0) | (fabsf(p.fy - 0.5f) > K.t1) | (fabsf(p.fz - 0.5f) > K.t2);
  p.base = 0;
  if (CLAMP || !TEX) {
    // O5 clamp: x <= 0 -> (0, f = 0), x >= n-1 -> (n-2, f = 1); exact floats (< 2^24)
    float ix = (float)x + flx, iy = (float)r.y + fly, iz = (float)r.z + flz;
    p.fx = ix < 0.f ? 0.f : (ix > V.fnx2 ? 1.f : p.fx);
    p.fy = iy < 0.f ? 0.f : (iy > V.fny2 ? 1.f : p.fy);
    p.fz = iz < 0.f ? 0.f : (iz > V.fnz2 ? 1.f : p.fz);
    ix = fminf(fmaxf(ix, 0.f), V.fnx2);
    iy = fminf(fmaxf(iy, 0.f), V.fny2);
    iz = fminf(fmaxf(iz, 0.f), V.fnz2);
    if (TEX) {
      p.u = ix + uoff;
      p.v = fmaf(iz, V.fnyp, iy) + V.voff;
    } else {
      p.base = ((int)iz * V.ny + (int)iy) * V.nx + (int)ix;
      p.u = p.v = 0.f;
    }
  } else {
    // gather x of corner x + flx of I_oth: (x + uoff) + flx; y: vrow + fma(flz, fnyp, fly)
    p.u = ((float)x + uoff) + flx;
    p.v = vrow + fmaf(flz, V.fnyp, fly);
  }
  return p;
}

// b = trilinear(I_oth, x) at a sample position (O5), positivity-exact lerps
template <bool TEX, class VT>
__device__ __forceinline__ float sample_b(const VT& V, const SamplePos& p, int side) {
  float c[8];
  if (TEX) gather2(V.texI, p.u, p.v, V.fnyp, c);
  else load8(side == 0 ? V.I[1] : V.I[0], p.base, V.nx, V.nx * V.ny, c);
  return tri8(c, p.fx, p.fy, p.fz, 1.f - p.fx, 1.f - p.fy, 1.f - p.fz);
}

// h of PAPER.md §4.1.2 (L318-322) with the case split (O6): a = I_side(q) exact,
// fg = "some contributing footprint corner is > 0"
__device__ __forceinline__ float h_of(float a, float b, bool fg) {
  if (a > 0.f && fg) {
    const float t = a - b;
    return t * t;
  }
  return (a == 0.f && !fg) ? 0.f : 1.f;
}

// The exact pass of a row (rare: some lane had an ambiguous sample).  Each such
// lane walks its own interval again, recomputes the same fp32 positions, and for
// its ambiguous samples decides fg exactly (int128 numerators, exact_fg) and
// adds h in fp64 (the main pass left them out).  Outside the sample loop, so
// the int128 code does not weigh on the loop's registers.
template <bool TEX, bool CLAMP, bool DUMP>
__device__ __noinline__ void exact_row(const VolLite V, const SampleK K, const RowCtx r, const LaneQ* LQ,
                                       bool pend, double2* accp, float* dump_h, unsigned char* dump_fg) {
  if (!pend) return;
  const int side = r.side;
  const float uoff = side ? V.uoffI[0] : V.uoffI[1];
  const long long rowlin = ((long long)r.z * V.ny + r.y) * V.nx;
  const uint2* __restrict__ own_row = V.own0 + (long long)side * V.V + rowlin;
  const float vrow = fmaf((float)r.z, V.fnyp, (float)r.y) + V.voff;
  double hs = 0.0;
  for (int x = r.xl; x <= r.xh; x++) {
    const SamplePos p = sample_pos<TEX, CLAMP>(V, K, r, x, (float)(x - r.xl), vrow, uoff);
    if (!p.amb) continue;
    const float b = sample_b<TEX>(V, p, side);
    const bool fg = exact_fg(LQ, side, x, r.y, r.z, p.dx, p.dy, p.dz, side == 0 ? V.I[1] : V.I[0], V.nx, V.ny,
                             V.nz);
    const float h = h_of(__uint_as_float(own_row[x].x), b, fg);
    hs += (double)h;
    if (DUMP) {
      dump_h[rowlin + x] = h;
      dump_fg[rowlin + x] = fg ? 1 : 0;
    }
  }
  accp->x += hs;
}

// a5 + a6 over one row: the warp walks x = X0..X1; lane l's sample is valid where
// x lies in its own interval.  TEX: gathers from the edge-padded textures; CLAMP:
// apply the O5 clamp (positions may leave the range the gather covers exactly).
// Ambiguous samples (O6 needs the exact decision) are left to exact_row.
// Returns the band entries of the lane's valid samples.
template <bool TEX, bool CLAMP, bool DUMP>
__device__ __forceinline__ int eval_row(const Volumes& V, const SampleK& K, const RowCtx& r, const LaneQ* LQ,
                                        double2* accp, float* dump_h, unsigned char* dump_fg) {
  const int side = r.side, oth = 1 - side;
  const float uoff = side ? V.uoffI[0] : V.uoffI[1];
  const long long rowlin = ((long long)r.z * V.ny + r.y) * V.nx;
  const float vrow = fmaf((float)r.z, V.fnyp, (float)r.y) + V.voff;
  // kf = x - xl (exact float); the lane's sample is valid iff 0 <= kf <= xh - xl
  const float kf0 = (float)(r.X0 - r.xl);
  const float lenf = (float)(r.xh - r.xl);
  unsigned pend = 0u;
  // ---- a5: h over the row.  a = I_side(q): one broadcast load per step.
  {
    const float* __restrict__ ap = (side ? V.I[1] : V.I[0]) + rowlin + r.X0;
    float kf = kf0;
    int x = r.X0;
    // fp32 partial sums per 16-voxel-aligned x block, then fp64: the grouping depends
    // only on the lane's own samples and absolute x, never on which solutions share
    // the warp (bitwise equal results for any sharding)
#pragma unroll 1
    while (x <= r.X1) {
      const int xe = min(r.X1, x | 15);
      float hf = 0.f;
      // two samples per iteration (x, x + 1): independent chains, four tld4 in flight;
      // hf still accumulates in x order
#pragma unroll 1
      for (; x < xe; x += 2, ap += 2) {
        const float a0 = __ldg(ap), a1 = __ldg(ap + 1);
        const float kf1 = kf + 1.0f;
        const bool v0 = (kf >= 0.f) & (kf <= lenf), v1 = (kf1 >= 0.f) & (kf1 <= lenf);
        const SamplePos p0 = sample_pos<TEX, CLAMP>(V, K, r, x, kf, vrow, uoff);
        const SamplePos p1 = sample_pos<TEX, CLAMP>(V, K, r, x + 1, kf1, vrow, uoff);
        kf += 2.0f;
        float b0, b1;
        if (TEX) {
          float c0[8], c1[8];
          gather2x2(V.texI, p0.u, p0.v, p1.u, p1.v, V.fnyp, c0, c1);
          b0 = tri8(c0, p0.fx, p0.fy, p0.fz, 1.f - p0.fx, 1.f - p0.fy, 1.f - p0.fz);
          b1 = tri8(c1, p1.fx, p1.fy, p1.fz, 1.f - p1.fx, 1.f - p1.fy, 1.f - p1.fz);
        } else {
          b0 = sample_b<TEX>(V, p0, side);
          b1 = sample_b<TEX>(V, p1, side);
        }
        const bool amb0 = v0 & p0.amb, amb1 = v1 & p1.amb;
        pend |= (amb0 | amb1) ? 1u : 0u;
        const float h0 = h_of(a0, b0, b0 > 0.f), h1 = h_of(a1, b1, b1 > 0.f);
        hf += (v0 & !amb0) ? h0 : 0.f;
        hf += (v1 & !amb1) ? h1 : 0.f;
        if (DUMP) {  // test hook morea_sample_map (one solution): the values just computed
          if (v0 && !amb0) { dump_h[rowlin + x] = h0; dump_fg[rowlin + x] = b0 > 0.f ? 1 : 0; }
          if (v1 && !amb1) { dump_h[rowlin + x + 1] = h1; dump_fg[rowlin + x + 1] = b1 > 0.f ? 1 : 0; }
        }
      }
      if (x == xe) {
        const float a = __ldg(ap);
        const bool valid = (kf >= 0.f) & (kf <= lenf);
        const SamplePos p = sample_pos<TEX, CLAMP>(V, K, r, x, kf, vrow, uoff);
        kf += 1.0f;
        const float b = sample_b<TEX>(V, p, side);
        const bool amb = valid & p.amb;
        pend |= amb ? 1u : 0u;
        const float h = h_of(a, b, b > 0.f);
        hf += (valid & !amb) ? h : 0.f;
        if (DUMP && valid && !amb) {
          dump_h[rowlin + x] = h;
          dump_fg[rowlin + x] = b > 0.f ? 1 : 0;
        }
        x++;
        ap++;
      }
      accp->x += (double)hf;
    }
  }
  // ---- a6: the guidance terms of the row's band voxels (runs of voxels with band
  // bits, precomputed per image row; the bits are warp-uniform): each lane gathers
  // the other side's maps at its own position
  int nb = 0;
  const long long rho = (long long)side * V.ny * V.nz + (long long)r.z * V.ny + r.y;
  const int q0 = __ldg(&V.run_off[rho]), q1 = __ldg(&V.run_off[rho + 1]);
  if (q0 < q1) {
    const float* __restrict__ drow = (side == 0 ? V.dmap[0] : V.dmap[1]) + rowlin;
    const uint2* __restrict__ orow = V.own[0] + (long long)side * V.V + rowlin;
    float gf = 0.f;
    int blk = -1;
#pragma unroll 1
    for (int q = q0; q < q1; q++) {
      const int2 run = __ldg(&V.runs[q]);
      const int xa = max(run.x, r.X0), xb = min(run.y, r.X1);
#pragma unroll 1
      for (int x = xa; x <= xb; x++) {
        if ((x >> 4) != blk) {  // same 16-voxel x blocks as h (deterministic grouping)
          accp->y += (double)gf;
          gf = 0.f;
          blk = x >> 4;
        }
        const float kf = kf0 + (float)(x - r.X0);
        const bool valid = (kf >= 0.f) & (kf <= lenf);
        const SamplePos p = sample_pos<TEX, CLAMP>(V, K, r, x, kf, vrow, uoff);
        unsigned m = __ldg(&orow[x].y);
        nb += valid ? __popc(m) : 0;
        while (m) {
          const int i = __ffs(m) - 1;
          m &= m - 1u;
          const float d = __ldg(drow + (long long)i * V.V + x);
          float e[8];
          if (TEX) {
            // map (oth, i) is volume oth K + i of texM; u carries oth fnxp already
            const float uu = fmaf((float)(oth * (V.K - 1) + i), V.fnxp, p.u);
            gather2(V.texM, uu, p.v, V.fnyp, e);
          } else {
            load8((oth == 0 ? V.dmap[0] : V.dmap[1]) + (long long)i * V.V, p.base, V.nx, V.nx * V.ny, e);
          }
          const float Dp = tri8(e, p.fx, p.fy, p.fz, 1.f - p.fx, 1.f - p.fy, 1.f - p.fz);
          const float dd = d - Dp;
          // O8: w_i (r - d)/r (d - D'(x))^2 where d < r (band bit); r - d as (r_f - d) + r_lo
          const float term = __ldg(&V.wfd[side * kMaxPairs + i]) * ((V.rf - d) + V.rlo) * (dd * dd);
          gf += valid ? term : 0.f;
        }
      }
    }
    accp->y += (double)gf;
  }
  if (__any_sync(FULLMASK, pend != 0u)) {
    VolLite vl;
    vl.nx = V.nx; vl.ny = V.ny; vl.nz = V.nz; vl.V = V.V;
    vl.fnx2 = V.fnx2; vl.fny2 = V.fny2; vl.fnz2 = V.fnz2; vl.fnyp = V.fnyp; vl.voff = V.voff;
    vl.uoffI[0] = V.uoffI[0]; vl.uoffI[1] = V.uoffI[1];
    vl.texI = V.texI;
    vl.I[0] = V.I[0]; vl.I[1] = V.I[1];
    vl.own0 = V.own[0];
    exact_row<TEX, CLAMP, DUMP>(vl, K, r, LQ, pend != 0u, accp, dump_h, dump_fg);
  }
  return nb;
}

// ---------------------------------------------------------------------------
// The sweep of one side of one item: union z range, per slice the lanes' y
// ranges, per row the lanes' exact x-intervals, then F::row over the union.
// ---------------------------------------------------------------------------
template <class F>
__device__ __forceinline__ void sweep_side(const Volumes& V, const SampleK& K, int side, int zb, int ze,
                                           const float4* __restrict__ slice, WarpLanes& L, const LaneQ* LQ,
                                           unsigned lane, F& f) {
  // slice fields: 0 fa[4], 1 fc[4], 2 vy[4], 3 vz[4], 4 (A02, A12, A22, d0x), 5 (d0y, d0z, lohi_y, lohi_z)
  const int flags = __float_as_int(slice[6 * 32 + lane].x);
  const bool has = (flags & 1) != 0;
  const int lhz = __float_as_int(slice[5 * 32 + lane].w);
  const int loz = lhz & 0xffff, hiz = lhz >> 16;
  const int zlo = max(loz, zb), zhi = min(hiz, ze - 1);
  const bool zany = has && zlo <= zhi;
  const int Z0 = __reduce_min_sync(FULLMASK, zany ? zlo : 0x7fffffff);
  const int Z1 = __reduce_max_sync(FULLMASK, zany ? zhi : (int)0x80000000);
  const bool regular_all = __all_sync(FULLMASK, !has || (flags & 4));
#pragma unroll 1
  for (int z = Z0; z <= Z1; z++) {
    int ylo = 1, yhi = 0;
    {
      const float4 s5 = slice[5 * 32 + lane];
      const int lhy = __float_as_int(s5.z);
      if (zany && z >= zlo && z <= zhi)
        slice_y_range(slice[2 * 32 + lane], slice[3 * 32 + lane], lhy & 0xffff, lhy >> 16, z, ylo, yhi);
      const float oz = (float)(z - loz);
      const float4 fa = slice[0 * 32 + lane], fc = slice[1 * 32 + lane], s4 = slice[4 * 32 + lane];
      // face crossings at (y = lo_y, z) and the displacement at (lo_x, lo_y, z)
      L.zb[lane] = make_float4(fmaf(fc.x, oz, fa.x), fmaf(fc.y, oz, fa.y), fmaf(fc.z, oz, fa.z),
                               fmaf(fc.w, oz, fa.w));
      L.zt[lane] = make_float4(fmaf(s4.x, oz, s4.w), fmaf(s4.y, oz, s5.x), fmaf(s4.z, oz, s5.y),
                               __int_as_float((ylo & 0xffff) | (yhi << 16)));
    }
    const int Y0 = __reduce_min_sync(FULLMASK, ylo <= yhi ? ylo : 0x7fffffff);
    const int Y1 = __reduce_max_sync(FULLMASK, ylo <= yhi ? yhi : (int)0x80000000);
#pragma unroll 1
    for (int y = Y0; y <= Y1; y++) {
      const float4 zt = lds4(&L.zt[lane]);
      const float4 k1 = lds4(&L.k1[lane]);
      const int yl = __float_as_int(zt.w) & 0xffff, yh = __float_as_int(zt.w) >> 16;
      const int lh = __float_as_int(k1.w);
      const int lox = lh & 1023, hix = (lh >> 10) & 1023, loy = (lh >> 20) & 1023;
      const bool rv = y >= yl && y <= yh && yl <= yh;
      const float oy = (float)(y - loy);
      int xl = 1, xh = 0;
      bool amb = false;
      if (regular_all) {
        // fast exact intervals: four fp32 crossings, the int64 decision only when a
        // crossing is within its error bound of an integer
        const float4 b = lds4(&L.zb[lane]), fb = lds4(&L.fb[lane]), th = lds4(&L.thr[lane]);
        const float flo = (float)lox - 4.5f, fhi = (float)hix + 4.5f;
        const float xs[4] = {fminf(fmaxf(fmaf(fb.x, oy, b.x), flo), fhi), fminf(fmaxf(fmaf(fb.y, oy, b.y), flo), fhi),
                             fminf(fmaxf(fmaf(fb.z, oy, b.z), flo), fhi), fminf(fmaxf(fmaf(fb.w, oy, b.w), flo), fhi)};
        const float tk[4] = {th.x, th.y, th.z, th.w};
        int l = lox, h = hix;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          amb = amb || (fabsf(xs[k] - rintf(xs[k])) <= fabsf(tk[k]));
          const int c = __float2int_ru(xs[k]);  // lower face: smallest x > x*; upper: largest x < x* = c - 1
          if (tk[k] > 0.f) l = max(l, c);
          else h = min(h, c - 1);
        }
        xl = l;
        xh = h;
        amb = amb && rv;
      } else {
        amb = rv;  // irregular item: every row of the lanes that have one is decided exactly
      }
      if (__any_sync(FULLMASK, amb)) {
        const int2 e = row_exact_if(amb, make_int2(xl, xh), LQ, side, y, z, lox, hix);
        xl = e.x;
        xh = e.y;
      }
      const bool ne = rv && xl <= xh;
      const int X0 = __reduce_min_sync(FULLMASK, ne ? xl : 0x7fffffff);
      const int X1 = __reduce_max_sync(FULLMASK, ne ? xh : (int)0x80000000);
      if (X0 > X1) continue;
      RowCtx r;
      r.side = side; r.z = z; r.y = y; r.X0 = X0; r.X1 = X1;
      r.xl = ne ? xl : 0x40000000;
      r.xh = ne ? xh : 0;
      const float ox = (float)((ne ? xl : lox) - lox);
      r.dx = fmaf(K.A00, ox, fmaf(k1.x, oy, zt.x));
      r.dy = fmaf(K.A10, ox, fmaf(k1.y, oy, zt.y));
      r.dz = fmaf(K.A20, ox, fmaf(k1.z, oy, zt.z));
      f.row(V, K, r, LQ, ne ? xh - xl + 1 : 0, L, lane);
    }
  }
}

// Build the lane's side state: slice fields to the warp's scratch (coalesced
// float4 [field][lane]), row fields to shared memory, per-sample in registers.
__device__ __forceinline__ void setup_side(const LaneQ& LQ, int side, bool ok, const Volumes& V, float4* slice,
                                           WarpLanes& L, unsigned lane, SampleK& K) {
  LaneFast G;
  if (ok) {
    int Q[4][3], Qo[4][3];
    lane_q(LQ, side, Q);
    lane_q(LQ, 1 - side, Qo);
    build_lane(Q, Qo, V.nx, V.ny, V.nz, G);
  } else {
    G.flags = 0;
  }
  if (!(G.flags & 1)) {
#pragma unroll
    for (int k = 0; k < 4; k++) { G.fa[k] = G.fb[k] = G.fc[k] = G.thr[k] = G.vy[k] = G.vz[k] = 0.f; }
#pragma unroll
    for (int a = 0; a < 3; a++) {
      G.d0[a] = G.eps[a] = 0.f;
      G.lo[a] = 1; G.hi[a] = 0;
#pragma unroll
      for (int b = 0; b < 3; b++) G.A[a][b] = 0.f;
    }
  }
  slice[0 * 32 + lane] = make_float4(G.fa[0], G.fa[1], G.fa[2], G.fa[3]);
  slice[1 * 32 + lane] = make_float4(G.fc[0], G.fc[1], G.fc[2], G.fc[3]);
  slice[2 * 32 + lane] = make_float4(G.vy[0], G.vy[1], G.vy[2], G.vy[3]);
  slice[3 * 32 + lane] = make_float4(G.vz[0], G.vz[1], G.vz[2], G.vz[3]);
  slice[4 * 32 + lane] = make_float4(G.A[0][2], G.A[1][2], G.A[2][2], G.d0[0]);
  slice[5 * 32 + lane] = make_float4(G.d0[1], G.d0[2], __int_as_float((G.lo[1] & 0xffff) | (G.hi[1] << 16)),
                                     __int_as_float((G.lo[2] & 0xffff) | (G.hi[2] << 16)));
  L.fb[lane] = make_float4(G.fb[0], G.fb[1], G.fb[2], G.fb[3]);
  L.thr[lane] = make_float4(G.thr[0], G.thr[1], G.thr[2], G.thr[3]);
  // empty lanes: lo = 1, hi = 0 on every axis (dims <= 768 < 1024: 10 bits each)
  L.k1[lane] = make_float4(G.A[0][1], G.A[1][1], G.A[2][1],
                           __int_as_float(G.lo[0] | (G.hi[0] << 10) | (G.lo[1] << 20)));
  slice[6 * 32 + lane] = make_float4(__int_as_float(G.flags), 0.f, 0.f, 0.f);
  K.A00 = G.A[0][0]; K.A10 = G.A[1][0]; K.A20 = G.A[2][0];
  K.t0 = 0.5f - G.eps[0]; K.t1 = 0.5f - G.eps[1]; K.t2 = 0.5f - G.eps[2];
}

// Row functors -----------------------------------------------------------------
template <bool TEX, bool DUMP>
struct EvalRow {
  bool clamp;  // warp-uniform per (item, side)
  float* dump_h;
  unsigned char* dump_fg;
  __device__ __forceinline__ int rows(const Volumes& V, const SampleK& K, const RowCtx& r, const LaneQ* LQ,
                                      double2* accp) {
    if (TEX) {
      if (clamp) return eval_row<true, true, DUMP>(V, K, r, LQ, accp, dump_h, dump_fg);
      return eval_row<true, false, DUMP>(V, K, r, LQ, accp, dump_h, dump_fg);
    }
    return eval_row<false, true, DUMP>(V, K, r, LQ, accp, dump_h, dump_fg);
  }
  __device__ __forceinline__ void row(const Volumes& V, const SampleK& K, const RowCtx& r, const LaneQ* LQ,
                                      int len, WarpLanes& L, unsigned lane) {
    // per-item counters of the lane (samples, side-0 samples); warp totals for profiling
    int2 c = L.cnt[lane];
    c.x += len;
    if (r.side == 0) c.y += len;
    L.cnt[lane] = c;
    const int nb = rows(V, K, r, LQ, &L.acc[lane]);
    const unsigned nbw = __reduce_add_sync(FULLMASK, (unsigned)nb);
    if (lane == 0) {
      L.nb += nbw;
      L.steps += r.X1 - r.X0 + 1;
    }
  }
};

// test hook / exports: visit every owned voxel of the lane
struct OwnerRow {  // owning tet per voxel, -2 = several owners
  int* owner;
  int tet;
  __device__ __forceinline__ void row(const Volumes& V, const SampleK&, const RowCtx& r, const LaneQ*, int,
                                      WarpLanes&, unsigned) {
    if (r.xl > r.xh) return;
    const long long b = ((long long)r.z * V.ny + r.y) * V.nx;
    for (int x = r.xl; x <= r.xh; x++) {
      const int old = atomicCAS(&owner[b + x], -1, tet);
      if (old != -1) atomicExch(&owner[b + x], -2);
    }
  }
};

struct MinOwnerRow {  // E3 pass 1: lowest owning tet id (deterministic under folds)
  int* owner;
  int tet;
  __device__ __forceinline__ void row(const Volumes& V, const SampleK&, const RowCtx& r, const LaneQ*, int,
                                      WarpLanes&, unsigned) {
    if (r.xl > r.xh) return;
    const long long b = ((long long)r.z * V.ny + r.y) * V.nx;
    for (int x = r.xl; x <= r.xh; x++) atomicMin(&owner[b + x], tet);
  }
};

// E1: label = 1 + lowest set bit of the object byte below M, 0 = no object
__device__ __forceinline__ int voxel_label(unsigned m, int M) {
  const unsigned v = m & ((1u << M) - 1u);
  return v ? __ffs(v) : 0;
}

struct LabelRow {
  const unsigned char* masks;
  int M;
  long long* counts;  // (M + 1) counters of this tet
  __device__ __forceinline__ void row(const Volumes& V, const SampleK&, const RowCtx& r, const LaneQ*, int,
                                      WarpLanes&, unsigned) {
    if (r.xl > r.xh) return;
    const long long b = ((long long)r.z * V.ny + r.y) * V.nx;
    for (int x = r.xl; x <= r.xh; x++)
      atomicAdd((unsigned long long*)&counts[voxel_label(__ldg(&masks[b + x]), M)], 1ull);
  }
};

// E3 pass 2: T(q) - q = sum_k e_k(q) U_k / (1024 |Delta|) (O4), exact numerator,
// one fp64 rounding (the oracle's operations), times the spacing, fp32
struct DvfRow {
  const int* owner;
  int tet;
  float* dvf;
  unsigned char* cov;
  __device__ __forceinline__ void row(const Volumes& V, const SampleK&, const RowCtx& r, const LaneQ* LQ, int,
                                      WarpLanes&, unsigned) {
    if (r.xl > r.xh) return;
    int Q[4][3], Qo[4][3];
    lane_q(*LQ, r.side, Q);
    lane_q(*LQ, 1 - r.side, Qo);
    ExactFaces F;
    exact_faces(Q, F);
    i64 det = det3(Q);
    if (det < 0) det = -det;
    const double den = __dmul_rn((double)det, 1024.0);
    const long long b = ((long long)r.z * V.ny + r.y) * V.nx;
    for (int x = r.xl; x <= r.xh; x++) {
      const long long lin = b + x;
      if (__ldg(&owner[lin]) != tet) continue;
      i64 e[4];
#pragma unroll
      for (int f = 0; f < 4; f++) e[f] = face_eval(F, f, x, r.y, r.z);
#pragma unroll
      for (int a = 0; a < 3; a++) {
        i128 n = 0;
#pragma unroll
        for (int f = 0; f < 4; f++) n += (i128)e[f] * (i128)(Qo[f][a] - Q[f][a]);
        const double u = __ddiv_rn((double)n, den);
        dvf[3LL * lin + a] = __double2float_rn(__dmul_rn(u, V.sp[a]));
      }
      cov[lin] = 1;
    }
  }
};

// ---------------------------------------------------------------------------
// Item decoding and the lane's tet vertices.
// ---------------------------------------------------------------------------
struct SweepItem {
  int v, slab, e, tet, sol, zb, ze;
  long long hgn;  // HGN index of the lane
};

__device__ __forceinline__ SweepItem decode_item(const EvalArgs& A, unsigned long long item, unsigned lane) {
  const int ng = (A.P + 31) >> 5;
  const long long per_v = (long long)A.n_slabs * ng;
  SweepItem it;
  it.v = (int)(item / (unsigned long long)per_v);
  const long long rem = (long long)item - (long long)it.v * per_v;
  const int sp = (int)(rem / ng);
  const int g = (int)(rem - (long long)sp * ng);
  it.slab = A.slab_sched[sp];
  it.e = A.slab_entry[it.slab];
  const int2 zz = A.slab_z[it.slab];
  it.zb = zz.x;
  it.ze = zz.y;
  it.tet = A.canon_tet ? A.canon_tet[it.e] : it.e;
  it.sol = g * 32 + (int)lane;
  it.hgn = ((long long)it.v * A.n_slabs + it.slab) * A.P + it.sol;
  return it;
}

// vectorised offset loads (3 x float2 per point, 24 B contiguous per lane)
__device__ __forceinline__ bool load_lane_q(const EvalArgs& A, const SweepItem& it, LaneQ& L) {
  const int4 tv = A.mesh.tets[it.tet];
  const int4 none = make_int4(-1, -1, -1, -1);
  const int4 slots = (it.v == 0 && A.canon_slots) ? A.canon_slots[it.e] : none;
  const int vid[4] = {tv.x, tv.y, tv.z, tv.w};
  const int sl[4] = {slots.x, slots.y, slots.z, slots.w};
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int j = vid[k];
    const float2* o = reinterpret_cast<const float2*>(
        sl[k] >= 0 ? A.new_vals + ((long long)it.sol * A.S_total + sl[k]) * 6
                   : A.offsets + ((long long)it.sol * A.mesh.N + j) * 6);
    const float2 o01 = __ldg(o), o23 = __ldg(o + 1), o45 = __ldg(o + 2);
    const float oo[6] = {o01.x, o01.y, o23.x, o23.y, o45.x, o45.y};
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const float b = __ldg(&A.mesh.base[3 * j + a]);
#pragma unroll
      for (int s = 0; s < 2; s++) {
        const i64 q = canon_q(b, oo[3 * s + a]);
        ok = ok && (q >= kQLo) && (q < kQHi);
        L.q[s][k][a] = (int)q;
      }
    }
  }
  return ok;
}

// ---------------------------------------------------------------------------
// k_sweep: persistent warps over the item queue (one block of kSweepWarps warps
// per SM; BlockQueue hands out consecutive items: the same slab for the next
// solution groups, so the block's footprints share L1).
// ---------------------------------------------------------------------------
template <bool TEX, bool DUMP>
__global__ void __launch_bounds__(kSweepThreads, 1) k_sweep(const EvalArgs A) {
  extern __shared__ __align__(16) unsigned char sweep_smem[];
  WarpLanes* lanes = reinterpret_cast<WarpLanes*>(sweep_smem);
  __shared__ BlockQueue bq;
  bq.init();
  unsigned warp, lane;
  asm volatile("shr.u32 %0, %1, 5;" : "=r"(warp) : "r"((unsigned)threadIdx.x));
  asm volatile("and.b32 %0, %1, 31;" : "=r"(lane) : "r"((unsigned)threadIdx.x));
  WarpScratch* ws = A.scratch + (long long)blockIdx.x * kSweepWarps + warp;
  float4* slice = &ws->slice[0][0];
  WarpLanes& L = lanes[warp];
  LaneQ* LQ = &ws->Q[lane];
  const int ng = (A.P + 31) >> 5;
  const long long n_items = (long long)A.n_raster_versions * A.n_slabs * ng;
  unsigned long long st_samples = 0, st_items = 0;
  if (lane == 0) L.nb = L.steps = 0;
  while (true) {
    const unsigned long long item = bq.claim(A.counter, (int)lane, n_items, MOREA_CLAIM_CHUNK, MOREA_CLAIM_SPREAD);
    if ((long long)item >= n_items) break;
    const SweepItem it = decode_item(A, item, lane);
    const bool active = it.sol < A.P;
    bool ok;
    {
      LaneQ q;
      ok = active && load_lane_q(A, it, q);
      *LQ = q;  // the lane's vertices, read back per side (not kept in registers)
    }
    EvalRow<TEX, DUMP> f;
    f.dump_h = A.dump_h;
    f.dump_fg = A.dump_fg;
    L.acc[lane] = make_double2(0.0, 0.0);
    L.cnt[lane] = make_int2(0, 0);
#pragma unroll 1
    for (int side = 0; side < 2; side++) {
      if (DUMP && side != A.dump_side) continue;
      SampleK K;
      __syncwarp();
      setup_side(*LQ, side, ok, A.vol, slice, L, lane, K);
      __syncwarp();
      const int fl = __float_as_int(slice[6 * 32 + lane].x);
      f.clamp = !__all_sync(FULLMASK, !(fl & 1) || (fl & ((TEX && kTexPad) ? 8 : 2)));
      sweep_side(A.vol, K, side, it.zb, it.ze, slice, L, LQ, lane, f);
    }
    __syncwarp();
    const int2 c = L.cnt[lane];
    if (active) {
      const double2 s = L.acc[lane];
      HGN out;
      out.h = s.x;
      out.g = s.y;
      out.n = c.x;
      out.n0 = c.y;
      A.hgn[it.hgn] = out;
    }
    st_samples += c.x;
    st_items += active ? 1 : 0;
  }
  if (A.stats) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      st_samples += __shfl_xor_sync(FULLMASK, st_samples, o);
      st_items += __shfl_xor_sync(FULLMASK, st_items, o);
    }
    if (lane == 0) {
      atomicAdd(&A.stats[0], st_samples);
      atomicAdd(&A.stats[1], L.nb);
      atomicAdd(&A.stats[2], st_items);
      atomicAdd(&A.stats[3], L.steps);
    }
  }
}

constexpr size_t kSweepDynSmem = sizeof(WarpLanes) * kSweepWarps;
// shared memory decides the L1/shared carve-out (steps 100, 132, ... KB, 1 KB per
// block reserved): at <= 99 KB the texture/L1 cache keeps 156 KB
static_assert(kSweepDynSmem + 1024 + 64 <= 100 * 1024, "k_sweep shared memory above the 100 KB carve-out step");

__global__ void k_owner_map(const EvalArgs A, int side, int* owner);
__global__ void k_min_owner(const EvalArgs A, int side, int* owner);
__global__ void k_dvf(const EvalArgs A, int side, const int* owner, float* dvf, unsigned char* cov);
__global__ void k_label_counts(const EvalArgs A, int side, const unsigned char* __restrict__ masks, int M,
                               long long* __restrict__ counts);

int sweep_blocks_per_sm(bool tex) {
  cudaFuncSetAttribute(k_sweep<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepDynSmem);
  cudaFuncSetAttribute(k_sweep<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepDynSmem);
  cudaFuncSetAttribute(k_sweep<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepDynSmem);
  cudaFuncSetAttribute(k_sweep<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepDynSmem);
  cudaFuncSetAttribute(k_owner_map, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepDynSmem);
  cudaFuncSetAttribute(k_min_owner, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepDynSmem);
  cudaFuncSetAttribute(k_dvf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepDynSmem);
  cudaFuncSetAttribute(k_label_counts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSweepDynSmem);
  int nb = 0;
  cudaError_t e = tex ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sweep<true, false>, kSweepThreads, kSweepDynSmem)
                      : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sweep<false, false>, kSweepThreads,
                                                                      kSweepDynSmem);
  if (e != cudaSuccess) return 1;
  return nb > 0 ? nb : 1;
}

int sweep_block_warps() { return kSweepWarps; }

cudaError_t launch_sweep(const EvalArgs& a, int grid, cudaStream_t s) {
  if (a.dump_h) {  // test hook morea_sample_map
    if (a.vol.use_tex) k_sweep<true, true><<<grid, kSweepThreads, kSweepDynSmem, s>>>(a);
    else k_sweep<false, true><<<grid, kSweepThreads, kSweepDynSmem, s>>>(a);
  } else {
    if (a.vol.use_tex) k_sweep<true, false><<<grid, kSweepThreads, kSweepDynSmem, s>>>(a);
    else k_sweep<false, false><<<grid, kSweepThreads, kSweepDynSmem, s>>>(a);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Exports and the owner-map test hook: the same per-lane geometry and row
// machinery (one solution: lane 0 of each warp; items = the slabs).
// ---------------------------------------------------------------------------
template <class F>
__device__ __forceinline__ void export_items(const EvalArgs& A, int side, F& f) {
  extern __shared__ __align__(16) unsigned char sweep_smem[];
  WarpLanes* lanes = reinterpret_cast<WarpLanes*>(sweep_smem);
  const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpScratch* ws = A.scratch + (long long)blockIdx.x * kSweepWarps + warp;
  float4* slice = &ws->slice[0][0];
  WarpLanes& L = lanes[warp];
  LaneQ* LQ = &ws->Q[lane];
  const long long n_items = (long long)A.n_slabs * ((A.P + 31) >> 5);
  for (long long item = (long long)blockIdx.x * kSweepWarps + warp; item < n_items;
       item += (long long)gridDim.x * kSweepWarps) {
    const SweepItem it = decode_item(A, (unsigned long long)item, lane);
    const bool active = it.sol < A.P;
    LaneQ q;
    const bool ok = active && load_lane_q(A, it, q);
    *LQ = q;
    SampleK K;
    __syncwarp();
    setup_side(q, side, ok, A.vol, slice, L, lane, K);
    __syncwarp();
    f.tet = it.tet;
    sweep_side(A.vol, K, side, it.zb, it.ze, slice, L, LQ, lane, f);
  }
}

__global__ void __launch_bounds__(kSweepThreads, 1) k_owner_map(const EvalArgs A, int side, int* owner) {
  OwnerRow f{owner, 0};
  export_items(A, side, f);
}

__global__ void __launch_bounds__(kSweepThreads, 1) k_min_owner(const EvalArgs A, int side, int* owner) {
  MinOwnerRow f{owner, 0};
  export_items(A, side, f);
}

__global__ void __launch_bounds__(kSweepThreads, 1) k_dvf(const EvalArgs A, int side, const int* owner,
                                                          float* dvf, unsigned char* cov) {
  DvfRow f{owner, 0, dvf, cov};
  export_items(A, side, f);
}

struct LabelRowT : LabelRow {
  int tet;
  long long* all;
  __device__ __forceinline__ void row(const Volumes& V, const SampleK& K, const RowCtx& r, const LaneQ* LQ,
                                      int len, WarpLanes& L, unsigned lane) {
    counts = all + (long long)tet * (M + 1);
    LabelRow::row(V, K, r, LQ, len, L, lane);
  }
};

__global__ void __launch_bounds__(kSweepThreads, 1) k_label_counts(const EvalArgs A, int side,
                                                                   const unsigned char* __restrict__ masks, int M,
                                                                   long long* __restrict__ counts) {
  LabelRowT f;
  f.masks = masks;
  f.M = M;
  f.counts = counts;
  f.all = counts;
  f.tet = 0;
  export_items(A, side, f);
}

__global__ void k_fill_int(int* p, long long n, int v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void k_fill_i64(long long* p, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = 0;
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

cudaError_t launch_owner_map(const EvalArgs& a, int grid, int side, int* owner, cudaStream_t s) {
  k_fill_int<<<1024, 256, 0, s>>>(owner, a.vol.V, -1);
  k_owner_map<<<grid, kSweepThreads, kSweepDynSmem, s>>>(a, side, owner);
  return cudaGetLastError();
}

cudaError_t launch_label_counts(const EvalArgs& a, int grid, int side, const unsigned char* masks, int M,
                                long long* counts, cudaStream_t s) {
  k_fill_i64<<<256, 256, 0, s>>>(counts, (long long)a.mesh.T * (M + 1));
  k_label_counts<<<grid, kSweepThreads, kSweepDynSmem, s>>>(a, side, masks, M, counts);
  return cudaGetLastError();
}

cudaError_t launch_dvf(const EvalArgs& a, int grid, int side, int* owner, float* dvf, unsigned char* cov,
                       cudaStream_t s) {
  k_fill_int<<<1024, 256, 0, s>>>(owner, a.vol.V, 0x7fffffff);
  cudaError_t e = cudaMemsetAsync(dvf, 0, (size_t)a.vol.V * 3 * sizeof(float), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(cov, 0, (size_t)a.vol.V, s);
  if (e != cudaSuccess) return e;
  k_min_owner<<<grid, kSweepThreads, kSweepDynSmem, s>>>(a, side, owner);
  k_dvf<<<grid, kSweepThreads, kSweepDynSmem, s>>>(a, side, owner, dvf, cov);
  return cudaGetLastError();
}

// morea_sobol_setup.cuh -- NEXT-1 (App. A.2): the k_setup part
// of the Sobol-in-tetrahedron sampler (seed, masks, sample count, fast-path error
// bound) and the exact -log routine (S5).  Included by morea_kernels.cu before
// k_setup; the sampling kernel is in morea_sobol.cuh.  Readings S1..S9: DESIGN.md §3.
// (Included inside namespace morea.)
#pragma once

// ---------------------------------------------------------------------------
// S3/S4: seed = FNV-1a (64 bit) over the 12 little-endian int32 Q.10 vertex
// coordinates of the sampled side; masks = high words of splitmix64(seed + j).
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long sb_splitmix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ unsigned long long sb_seed(const int Q[4][3]) {
  unsigned long long h = 14695981039346656037ULL;
#pragma unroll
  for (int k = 0; k < 4; k++)
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const unsigned c = (unsigned)Q[k][a];
#pragma unroll
      for (int b = 0; b < 4; b++) {
        h ^= (c >> (8 * b)) & 0xFFu;
        h *= 1099511628211ULL;
      }
    }
  return h;
}

// S5: log r (r > 0) by the fixed operation sequence both implementations use
// (frexp, one division, degree-23 odd series, split ln 2); explicit _rn
// intrinsics so that nothing is contracted into an FMA.  -log((x + 1/2) 2^-32)
// is the Sobol sampler's exponential variate; the repair's Gaussian draws use
// the same routine.
__device__ __noinline__ double sb_det_ln(double r) {
  int e;
  double m = frexp(r, &e);
  if (m < 0.70710678118654752440) {
    m = __dmul_rn(m, 2.0);
    e = e - 1;
  }
  const double t = __ddiv_rn(__dadd_rn(m, -1.0), __dadd_rn(m, 1.0));
  const double t2 = __dmul_rn(t, t);
  const double c[12] = {1.0 / 23.0, 1.0 / 21.0, 1.0 / 19.0, 1.0 / 17.0, 1.0 / 15.0, 1.0 / 13.0,
                        1.0 / 11.0, 1.0 / 9.0,  1.0 / 7.0,  1.0 / 5.0,  1.0 / 3.0,  1.0};
  double p = c[0];
#pragma unroll
  for (int i = 1; i < 12; i++) p = __dadd_rn(__dmul_rn(p, t2), c[i]);
  const double lm = __dmul_rn(__dmul_rn(2.0, t), p);
  const double de = (double)e;
  return __dadd_rn(__dmul_rn(de, 6.93147180369123816490e-01),
                   __dadd_rn(__dmul_rn(de, 1.90821492927058770002e-10), lm));
}

__device__ __forceinline__ double sb_neg_log(unsigned x) {
  return -sb_det_ln(__dmul_rn(__dadd_rn((double)x, 0.5), 2.3283064365386963e-10));
}

// ---------------------------------------------------------------------------
// k_setup part (S3, S4, S6 and the fast-path error bound)
// ---------------------------------------------------------------------------
__device__ void build_sobol(const int Q[4][3], const int Qo[4][3], const Volumes& V, double rate,
                            SobolRec& R) {
  const i64 det = det3(Q);
  const i64 absdet = det < 0 ? -det : det;
  // S6: N = floor(rate |Delta| / (6 1024^3) + 1/2) with the oracle's operations
  const double scale = __ddiv_rn(rate, 6442450944.0);
  R.N = (long long)floor(__dadd_rn(__dmul_rn((double)absdet, scale), 0.5));
  const unsigned long long seed = sb_seed(Q);
#pragma unroll
  for (int j = 0; j < 4; j++) R.mask[j] = (unsigned)(sb_splitmix64(seed + (unsigned long long)j) >> 32);
  const int dims[3] = {V.nx, V.ny, V.nz};
  bool inside = true;    // every vertex of both sides in [0, n-1]
  bool inside_p = true;  // ... in [-1 + 1/16, n - 1/16]: no clamp on the edge-padded textures
  float dmax = 0.f;
#pragma unroll
  for (int k = 0; k < 4; k++)
#pragma unroll
    for (int a = 0; a < 3; a++) {
      R.Q[k][a] = Q[k][a];
      R.Qo[k][a] = Qo[k][a];
      inside = inside && Q[k][a] >= 0 && Q[k][a] <= 1024 * (dims[a] - 1) && Qo[k][a] >= 0 &&
               Qo[k][a] <= 1024 * (dims[a] - 1);
      inside_p = inside_p && Q[k][a] >= -1024 + 64 && Q[k][a] <= 1024 * dims[a] - 64 &&
                 Qo[k][a] >= -1024 + 64 && Qo[k][a] <= 1024 * dims[a] - 64;
    }
#pragma unroll
  for (int a = 0; a < 3; a++) {
    // X_0 = i0 + x0 with i0 = floor(X_0): the fp32 position is accumulated around
    // x0 in [0, 1), so its rounding is relative to the tet size, not to |X|
    R.i0[a] = (float)(Q[0][a] >> 10);
    R.i0o[a] = (float)(Qo[0][a] >> 10);
    R.x0[a] = (float)(Q[0][a] & 1023) * (1.0f / 1024.0f);
    R.x0o[a] = (float)(Qo[0][a] & 1023) * (1.0f / 1024.0f);
#pragma unroll
    for (int k = 1; k < 4; k++) {
      R.D[k - 1][a] = (float)(Q[k][a] - Q[0][a]) * (1.0f / 1024.0f);
      R.Do[k - 1][a] = (float)(Qo[k][a] - Qo[0][a]) * (1.0f / 1024.0f);
      dmax = fmaxf(dmax, fmaxf(fabsf(R.D[k - 1][a]), fabsf(R.Do[k - 1][a])));
    }
  }
  // Error of the fp32 offset y = x0 + sum_k l_k D_k against the oracle's position
  // (DESIGN.md §4.5): e_j = -lg2.approx(u_j) (absolute error <= 2^-22.6, the
  // exponent part is exact) on u_j rounded to fp32 (2^-24 relative, 2^-23.47 in
  // e_j): Delta = sum_j |de_j| <= 2^-20; lambda_j = e_j rcp_rn(s) with s summed in
  // fp32: sum_k |dl_k| <= 2 Delta / s + 2^-21; three fma roundings
  // <= 1.5 2^-23 (1 + 3 D).  eps = 2x the bound, as epsA / s + epsB.
  R.epsA = 2.0f * dmax * 0x1.0p-19f;
  R.epsB = 2.0f * (dmax * 0x1.0p-21f + 1.5f * 0x1.0p-23f * (1.0f + 3.0f * dmax));
  R.flags = (R.N > 0 ? 1 : 0) | (inside ? 2 : 0) | (inside_p ? 4 : 0);
  R.pad = 0;
}

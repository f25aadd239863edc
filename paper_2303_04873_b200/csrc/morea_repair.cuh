// morea_repair.cuh -- NEXT-2: batched fold repair (§4.3.1) on
// sm_100a, included by morea_kernels.cu (one TU, inside namespace morea).
//
// "For each point in a folded tetrahedron, the method mutates the point using a
// Gaussian distribution scaled by its estimated distance to the surrounding 3D
// polygon.  After 64 samples, the change with the best constraint improvement
// is selected, if present.  If all samples result in a deterioration, repair is
// aborted."  Readings P1..P8: DESIGN.md §3.
//
// One 64-thread block per solution: the points of a solution are repaired in
// sequence (each accepted move changes the next point's neighbourhood), the 64
// candidates of a point in parallel, one per thread.  Every score is exact
// (int64 determinants) and every floating-point step follows the oracle's
// operation order with _rn intrinsics, so the chosen candidate and the written
// offsets are bit-identical to the oracle's.
// (Included inside namespace morea.)
#pragma once

constexpr int kRepairCandidates = 64;

struct RepairArgs {
  MeshDev mesh;
  double sp[3];
  int P;
  long long sol_base;            // global index of solution 0 (generator key, sharding)
  float* offsets;                // P*N*6, updated in place
  const unsigned char* fixed;    // N*3 or nullptr (P8)
  const int* inc_off;            // incidence CSR (ascending tet ids)
  const int* inc;
  unsigned long long seed;
  int* moved;                    // P
  int* aborted;                  // P
};

// P5: Marsaglia polar pair from splitmix64(key + ctr), det_ln for ln s
__device__ __forceinline__ void rp_gauss_pair(unsigned long long key, unsigned long long& ctr,
                                              double& z0, double& z1) {
  for (;;) {
    const unsigned long long w = sb_splitmix64(key + ctr++);
    const double u =
        __dadd_rn(__dmul_rn(__dadd_rn((double)(unsigned)(w >> 32), 0.5), 4.656612873077392578125e-10), -1.0);
    const double v =
        __dadd_rn(__dmul_rn(__dadd_rn((double)(unsigned)w, 0.5), 4.656612873077392578125e-10), -1.0);
    const double sq = __dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v));
    if (!(sq < 1.0) || sq == 0.0) continue;
    const double f = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, sb_det_ln(sq)), sq));
    z0 = __dmul_rn(u, f);
    z1 = __dmul_rn(v, f);
    return;
  }
}

__device__ __forceinline__ unsigned long long rp_key(unsigned long long seed, long long k, int s, int j,
                                                     int c) {
  unsigned long long h = sb_splitmix64(seed + (unsigned long long)k);
  h = sb_splitmix64(h + (unsigned long long)s);
  h = sb_splitmix64(h + (unsigned long long)j);
  return sb_splitmix64(h + (unsigned long long)c);
}

// Q of the 4 vertices of tet t on side s; point j's side-s offset replaced by o3 (j >= 0)
__device__ __forceinline__ bool rp_tet_coords(const RepairArgs& A, const float* off, int t, int s, int j,
                                              const float o3[3], int Q[4][3]) {
  const int4 tv = A.mesh.tets[t];
  const int vid[4] = {tv.x, tv.y, tv.z, tv.w};
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 4; k++) {
    const int v = vid[k];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const float o = (v == j) ? o3[a] : off[6 * v + 3 * s + a];
      const long long q = canon_q(__ldg(&A.mesh.base[3 * v + a]), o);
      ok = ok && q >= kQLo && q < kQHi;
      Q[k][a] = (int)q;
    }
  }
  return ok;
}

struct RpScore {
  int folds;
  double sev;
};

__device__ __forceinline__ bool rp_less(const RpScore& a, const RpScore& b) {
  return a.folds < b.folds || (a.folds == b.folds && a.sev < b.sev);
}

// P6: (folded incident tets, their severity) of point j on side s with offset o3
__device__ RpScore rp_score(const RepairArgs& A, const float* off, int s, int j, const float o3[3]) {
  RpScore r{0, 0.0};
  for (int u = A.inc_off[j]; u < A.inc_off[j + 1]; u++) {
    const int t = A.inc[u];
    int Q[4][3];
    if (!rp_tet_coords(A, off, t, s, j, o3, Q)) return RpScore{0x7fffffff, __longlong_as_double(0x7ff0000000000000LL)};
    const long long d = det3(Q);
    const int sg = (d > 0) - (d < 0);
    if (sg != A.mesh.ref[t]) {
      r.folds++;
      // |Delta| / (6 1024^3) sp_x sp_y sp_z in the oracle's order
      const double sv = __dmul_rn(__dmul_rn(__dmul_rn(__ddiv_rn((double)(d < 0 ? -d : d), 6442450944.0),
                                                      A.sp[0]), A.sp[1]), A.sp[2]);
      r.sev = __dadd_rn(r.sev, sv);
    }
  }
  return r;
}

// P4: sigma = 1/2 min over incident tets (unfolded ones, else all) of |Delta| / (1024 |n_opp|)
__device__ double rp_sigma(const RepairArgs& A, const float* off, int s, int j) {
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  double best_unf = inf, best_all = inf;
  for (int u = A.inc_off[j]; u < A.inc_off[j + 1]; u++) {
    const int t = A.inc[u];
    int Q[4][3];
    if (!rp_tet_coords(A, off, t, s, -1, nullptr, Q)) continue;
    const int4 tv = A.mesh.tets[t];
    const int vid[4] = {tv.x, tv.y, tv.z, tv.w};
    int kj = 0;
    for (int k = 0; k < 4; k++)
      if (vid[k] == j) kj = k;
    int f[3], m = 0;
    for (int k = 0; k < 4; k++)
      if (k != kj) f[m++] = k;
    double e1[3], e2[3];
    for (int a = 0; a < 3; a++) {
      e1[a] = (double)(Q[f[1]][a] - Q[f[0]][a]);
      e2[a] = (double)(Q[f[2]][a] - Q[f[0]][a]);
    }
    const double n0 = __dsub_rn(__dmul_rn(e1[1], e2[2]), __dmul_rn(e1[2], e2[1]));
    const double n1 = __dsub_rn(__dmul_rn(e1[2], e2[0]), __dmul_rn(e1[0], e2[2]));
    const double n2 = __dsub_rn(__dmul_rn(e1[0], e2[1]), __dmul_rn(e1[1], e2[0]));
    const double nn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(n0, n0), __dmul_rn(n1, n1)), __dmul_rn(n2, n2)));
    if (!(nn > 0.0)) continue;
    const long long d = det3(Q);
    const double dist = __ddiv_rn((double)(d < 0 ? -d : d), __dmul_rn(nn, 1024.0));
    if (dist < best_all) best_all = dist;
    if (((d > 0) - (d < 0)) == A.mesh.ref[t] && dist < best_unf) best_unf = dist;
  }
  const double b = best_unf < inf ? best_unf : best_all;
  return b < inf ? __dmul_rn(0.5, b) : 0.5;
}

__global__ void __launch_bounds__(kRepairCandidates) k_repair(const RepairArgs A) {
  extern __shared__ unsigned char pts[];  // N flags
  __shared__ int s_fold[kRepairCandidates];
  __shared__ double s_sev[kRepairCandidates];
  __shared__ int s_best;
  const int tid = threadIdx.x;
  const int sol = blockIdx.x;
  const int N = A.mesh.N, T = A.mesh.T;
  float* off = A.offsets + (long long)sol * N * 6;
  int moved = 0, aborted = 0;
  for (int s = 0; s < 2; s++) {
    // P1/P2: vertices of the tets folded on side s at the start of the pass
    for (int j = tid; j < N; j += blockDim.x) pts[j] = 0;
    __syncthreads();
    for (int t = tid; t < T; t += blockDim.x) {
      int Q[4][3];
      if (!rp_tet_coords(A, off, t, s, -1, nullptr, Q)) continue;
      const long long d = det3(Q);
      if (((d > 0) - (d < 0)) != A.mesh.ref[t]) {
        const int4 tv = A.mesh.tets[t];
        pts[tv.x] = 1; pts[tv.y] = 1; pts[tv.z] = 1; pts[tv.w] = 1;
      }
    }
    __syncthreads();
    for (int j = 0; j < N; j++) {
      if (!pts[j]) continue;  // block-uniform
      float cur[3];
      for (int a = 0; a < 3; a++) cur[a] = off[6 * j + 3 * s + a];
      const RpScore s0 = rp_score(A, off, s, j, cur);
      if (s0.folds == 0) continue;  // P3
      const double sigma = rp_sigma(A, off, s, j);
      // P5: candidate tid
      double z[3], zd;
      unsigned long long ctr = 0;
      const unsigned long long key = rp_key(A.seed, A.sol_base + sol, s, j, tid);
      rp_gauss_pair(key, ctr, z[0], z[1]);
      rp_gauss_pair(key, ctr, z[2], zd);
      float o3[3];
      for (int a = 0; a < 3; a++)
        o3[a] = (A.fixed && A.fixed[3 * j + a]) ? cur[a]
                                                : __double2float_rn(__dadd_rn((double)cur[a], __dmul_rn(sigma, z[a])));
      const RpScore sc = rp_score(A, off, s, j, o3);
      s_fold[tid] = sc.folds;
      s_sev[tid] = sc.sev;
      __syncthreads();
      if (tid == 0) {  // P7: lexicographic minimum, lowest index on ties
        int b = 0;
        for (int c = 1; c < kRepairCandidates; c++)
          if (s_fold[c] < s_fold[b] || (s_fold[c] == s_fold[b] && s_sev[c] < s_sev[b])) b = c;
        const RpScore bs{s_fold[b], s_sev[b]};
        s_best = rp_less(bs, s0) ? b : -1;
      }
      __syncthreads();
      if (s_best == tid)
        for (int a = 0; a < 3; a++) off[6 * j + 3 * s + a] = o3[a];
      if (s_best >= 0) moved++;
      else aborted++;
      __syncthreads();
    }
  }
  if (tid == 0) {
    if (A.moved) A.moved[sol] = moved;
    if (A.aborted) A.aborted[sol] = aborted;
  }
}

cudaError_t launch_repair(const MeshDev& m, const double sp[3], int P, long long sol_base, float* offsets,
                          const unsigned char* fixed, const int* inc_off, const int* inc,
                          unsigned long long seed, int* moved, int* aborted, cudaStream_t s) {
  if (P <= 0) return cudaSuccess;
  RepairArgs A;
  A.mesh = m;
  for (int a = 0; a < 3; a++) A.sp[a] = sp[a];
  A.P = P;
  A.sol_base = sol_base;
  A.offsets = offsets;
  A.fixed = fixed;
  A.inc_off = inc_off;
  A.inc = inc;
  A.seed = seed;
  A.moved = moved;
  A.aborted = aborted;
  k_repair<<<P, kRepairCandidates, (size_t)m.N, s>>>(A);
  return cudaGetLastError();
}

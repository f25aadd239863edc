// morea_mix.cuh -- NEXT-3: device-side optimal mixing of one FOS colour class
// (§3) on sm_100a, included by morea_kernels.cu (inside
// namespace morea).
//
// "Variation then proceeds by considering variables in FOS elements jointly in a
// procedure called optimal mixing.  In this step, distributions are estimated for
// each FOS element in each cluster, and new, partial solutions are sampled from
// these distributions.  Newly sampled partial solutions are evaluated and
// accepted if their insertion into the parent solution results in a solution
// that dominates the parent solution or that is non-dominated in the current
// elitist archive."  Readings M1..M7: DESIGN.md §3.
//
// One call = sample (k_mix_sample) -> partial evaluation of every (solution,
// group) against the class-start state with the per-tet cache (the a8 path) ->
// per-solution acceptance scan in group order (k_mix_accept; the groups of a
// colour class have disjoint dependent tets, so each group's delta is independent
// of the others and only the acceptance is sequential) -> commit of the accepted
// offsets and cache rows (k_mix_commit).  No host round trip.
// (Included inside namespace morea.)
#pragma once

constexpr int kMixMaxDim = 192;  // 6 * 32 points per FOS element


__device__ __forceinline__ unsigned long long mix_key(unsigned long long seed, long long gen, long long k,
                                                      int g) {
  unsigned long long h = sb_splitmix64(seed + (unsigned long long)gen);
  h = sb_splitmix64(h + (unsigned long long)k);
  return sb_splitmix64(h + (unsigned long long)g);
}

// M1-M3: one thread per (solution, group)
__global__ void k_mix_sample(const MixArgs A) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)A.P * A.G) return;
  const int k = (int)(i / A.G), g = (int)(i % A.G);
  const int s0 = A.grp_off[g], ns = A.grp_off[g + 1] - s0;
  const int d = 6 * ns;
  const int c = A.cluster[k];
  const double* mu = A.mu + (long long)c * A.mu_stride + A.model_off[2 * g];
  const double* L = A.L + (long long)c * A.L_stride + A.model_off[2 * g + 1];
  double z[kMixMaxDim];
  unsigned long long ctr = 0;
  const unsigned long long key = mix_key(A.seed, A.gen, A.sol_base + k, g);
  for (int j = 0; j < d; j += 2) rp_gauss_pair(key, ctr, z[j], z[j + 1]);
  for (int v = 0; v < d; v++) {
    double x = mu[v];
    for (int j = 0; j <= v; j++) x = __dadd_rn(x, __dmul_rn(L[(long long)v * d + j], z[j]));
    const int pt = A.changed[s0 + v / 6], cc = v % 6;
    const float parent = A.offsets[((long long)k * A.N + pt) * 6 + cc];
    A.new_vals[((long long)k * A.S_total + s0 + v / 6) * 6 + cc] =
        (A.fixed && A.fixed[3 * pt + cc % 3]) ? parent : __double2float_rn(x);
  }
}

__device__ __forceinline__ bool mix_dominates(const double a[3], const double b[3]) {
  bool better = false;
#pragma unroll
  for (int i = 0; i < 3; i++) {
    if (a[i] > b[i]) return false;
    if (a[i] < b[i]) better = true;
  }
  return better;
}

// M4-M6: one thread per solution, groups in id order.  cand = current + (pacc_g - base).
__global__ void k_mix_accept(int P, int G, int T, const morea_acc* __restrict__ base,
                             const morea_acc* __restrict__ pacc, morea_acc* __restrict__ acc,
                             double* __restrict__ obj, const double* __restrict__ archive, int A_n,
                             double steer_max, unsigned char* __restrict__ accepted) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= P) return;
  const morea_acc b = base[k];
  morea_acc cur = b;
  double co[3] = {obj[3 * k], obj[3 * k + 1], obj[3 * k + 2]};
  for (int g = 0; g < G; g++) {
    const morea_acc p = pacc[(long long)k * G + g];
    morea_acc cand;
    cand.h_sum = cur.h_sum + (p.h_sum - b.h_sum);
    cand.g_sum = cur.g_sum + (p.g_sum - b.g_sum);
    cand.m_sum = cur.m_sum + (p.m_sum - b.m_sum);
    cand.severity = cur.severity + (p.severity - b.severity);
    cand.n_samples = cur.n_samples + (p.n_samples - b.n_samples);
    cand.folds = cur.folds + (p.folds - b.folds);
    cand.flags = (cur.flags & MOREA_F_DOMAIN) | (p.flags & MOREA_F_DOMAIN);
    if (cand.n_samples == 0) cand.flags |= MOREA_F_EMPTY;
    bool ok = cand.folds == 0 && !(cand.flags & (MOREA_F_DOMAIN | MOREA_F_EMPTY));  // M4
    double o[3] = {0.0, 0.0, 0.0};
    if (ok) {
      o[0] = cand.m_sum / (10.0 * (double)T);
      o[1] = cand.h_sum / (double)cand.n_samples;
      o[2] = cand.g_sum / (double)cand.n_samples;
      if (steer_max > 0.0 && !(o[2] <= steer_max)) ok = false;  // M5 steering bound
    }
    if (ok && !mix_dominates(o, co)) {  // M5: else not dominated by any archive member
      for (int a = 0; a < A_n && ok; a++) {
        const double ar[3] = {archive[3 * a], archive[3 * a + 1], archive[3 * a + 2]};
        if (mix_dominates(ar, o)) ok = false;
      }
    }
    if (accepted) accepted[(long long)k * G + g] = ok ? 1 : 0;
    if (ok) {  // M6
      cur = cand;
      co[0] = o[0]; co[1] = o[1]; co[2] = o[2];
    }
  }
  acc[k] = cur;
  obj[3 * k] = co[0]; obj[3 * k + 1] = co[1]; obj[3 * k + 2] = co[2];
}

// commit: accepted groups' point values and the new per-tet cache rows
__global__ void k_mix_commit(int P, int G, int N, int T, int S_total, int n_entries,
                             const unsigned char* __restrict__ accepted, const int* __restrict__ grp_off,
                             const int* __restrict__ changed, const int* __restrict__ group_off,
                             const int* __restrict__ canon_tet, const float* __restrict__ new_vals,
                             const double* __restrict__ dep_cache, float* __restrict__ offsets,
                             double* __restrict__ tet_cache) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= (long long)P * G) return;
  const int k = (int)(w / G), g = (int)(w % G);
  if (!accepted[w]) return;
  for (int i = grp_off[g] * 6 + lane; i < grp_off[g + 1] * 6; i += 32) {
    const int pt = changed[i / 6];
    offsets[((long long)k * N + pt) * 6 + i % 6] = new_vals[((long long)k * S_total) * 6 + i];
  }
  for (int i = group_off[g] * 4 + lane; i < group_off[g + 1] * 4; i += 32) {
    const int e = i / 4;
    tet_cache[((long long)k * T + canon_tet[e]) * 4 + i % 4] = dep_cache[((long long)k * n_entries) * 4 + i];
  }
}

cudaError_t launch_mix_sample(const MixArgs& a, cudaStream_t s) {
  const long long n = (long long)a.P * a.G;
  if (n == 0) return cudaSuccess;
  k_mix_sample<<<(unsigned)((n + 63) / 64), 64, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_mix_accept(int P, int G, int T, const morea_acc* base, const morea_acc* pacc, morea_acc* acc,
                              double* obj, const double* archive, int A_n, double steer_max,
                              unsigned char* accepted, cudaStream_t s) {
  if (P == 0) return cudaSuccess;
  k_mix_accept<<<(P + 127) / 128, 128, 0, s>>>(P, G, T, base, pacc, acc, obj, archive, A_n, steer_max,
                                               accepted);
  return cudaGetLastError();
}

cudaError_t launch_mix_commit(int P, int G, int N, int T, int S_total, int n_entries,
                              const unsigned char* accepted, const int* grp_off, const int* changed,
                              const int* group_off, const int* canon_tet, const float* new_vals,
                              const double* dep_cache, float* offsets, double* tet_cache, cudaStream_t s) {
  const long long n = (long long)P * G * 32;
  if (n == 0) return cudaSuccess;
  k_mix_commit<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P, G, N, T, S_total, n_entries, accepted, grp_off,
                                                           changed, group_off, canon_tet, new_vals, dep_cache,
                                                           offsets, tet_cache);
  return cudaGetLastError();
}

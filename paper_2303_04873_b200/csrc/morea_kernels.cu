// morea_kernels.cu -- sm_100a kernels of the MOREA hot path (arXiv 2303.04873).
//
// Rows of SURVEY.md §8(a) and where they live:
//   a0 load-time maps          k_distance_maps, k_band_mask, k_validate_volume
//   a1 genotype decode          canon_q (fp64, exact Q.10 rounding)
//   a2 per-tet geometry + fold  k_setup (folds, severity, magnitude per item);
//                               build_lane in k_sweep (per-lane fast geometry)
//   a3 magnitude                k_setup (magnitude)
//   a4 ownership rasterizer     k_sweep: per-lane exact row intervals (morea_sweep.cuh)
//   a5 map + sample + h         k_sweep: eval_row (exact case split, exact_fg)
//   a6 guidance term            k_sweep: eval_row (warp-uniform band bits, in place)
//   a7 reductions               per-lane sums in k_sweep, fixed-order k_reduce
//   a8 partial evaluation       version 0/1 items + k_reduce with base_acc
//   a9 fold check               k_check_folds
// The readings of the paper (O1..O13) are cited per function.
//
// Work decomposition.  k_setup: one thread per (version, tet,
// solution) computes the per-tet scalar terms (folds, severity, magnitude).
// k_sweep: one 28-warp block per SM pulls items (version, tet z-slab, group of
// 32 solutions) from a global queue; lane l of a warp evaluates solution
// 32 g + l, the warp walking the union of the lanes' lattice rows (see
// morea_sweep.cuh).  Further sm_100a kernels: morea_sobol*.cuh (NEXT-1 Sobol
// sampler), morea_repair.cuh (NEXT-2 fold repair), morea_mix.cuh (NEXT-3 optimal
// mixing), morea_sweep.cuh exports (NEXT-4 object counts and DVF).
#include <cuda_runtime.h>

#include <cstdint>

#include "morea.h"
#include "morea_internal.h"

#ifndef MOREA_SOBOL_WARPS
#define MOREA_SOBOL_WARPS 28  // k_sobol: warps of its one block per SM
#endif

#ifndef MOREA_CLAIM_CHUNK
#define MOREA_CLAIM_CHUNK 112  // k_sweep, k_sobol: at most this many items per global claim of BlockQueue
#endif

#ifndef MOREA_CLAIM_SPREAD
#define MOREA_CLAIM_SPREAD 16  // k_sweep, k_sobol: at least this many claims per block per launch where possible
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
// k_setup: one thread per (version, canonical entry, solution): the per-tet
// scalar terms (folds, severity, magnitude, domain flag); in Sobol mode also the
// SobolRec of each side.  (The voxel-centre sweep builds its geometry per lane.)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_setup(const EvalArgs A) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per_v = (long long)A.n_entries * A.P;
  if (i >= per_v * A.n_setup_versions) return;
  const int v = (int)(i / per_v);
  const long long rem = i - (long long)v * per_v;
  const int e = (int)(rem / A.P);
  const int sol = (int)(rem - (long long)e * A.P);
  const int tet = A.canon_tet ? A.canon_tet[e] : e;
  const int4 none = make_int4(-1, -1, -1, -1);
  const int4 slots = (v == 0 && A.canon_slots) ? A.canon_slots[e] : none;
  int Q[2][4][3];
  Scal sc;
  sc.m = sc.sev = 0.0;
  sc.folds = sc.flags = 0;
  sc.pad[0] = sc.pad[1] = 0;
  const bool sobol = A.sampler == 1 && v < A.n_raster_versions;
  if (!load_tet(A, sol, A.mesh.tets[tet], slots, Q)) {
    sc.flags = 1;  // domain: the tet contributes nothing
    A.scal[i] = sc;
    if (sobol) {
      A.sgeom[2 * i].flags = 0;
      A.sgeom[2 * i + 1].flags = 0;
    }
    return;
  }
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
  if (!sobol) {
    A.scal[i] = sc;
    return;
  }
#pragma unroll 1
  for (int s = 0; s < 2; s++) {
    SobolRec G;
    build_sobol(Q[s], Q[1 - s], V, A.rate, G);
    if (G.N > 0x7fffffffLL) {  // beyond the 32-bit point counter: flagged like a domain
      sc.flags = 1;            // error (objectives NaN), the side contributes nothing
      G.flags = 0;
    }
    const int4* src = reinterpret_cast<const int4*>(&G);
    int4* dst = reinterpret_cast<int4*>(&A.sgeom[2 * i + s]);
#pragma unroll
    for (int t = 0; t < (int)(sizeof(SobolRec) / 16); t++) dst[t] = src[t];
  }
  A.scal[i] = sc;
}

cudaError_t launch_setup(const EvalArgs& a, cudaStream_t s) {
  const long long n = (long long)a.n_setup_versions * a.n_entries * a.P;
  if (n == 0) return cudaSuccess;
  k_setup<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(a);
  return cudaGetLastError();
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

#include "morea_sweep.cuh"

// per-tet sums of one (version, entry, solution): its z-slabs in order
__device__ __forceinline__ HGN hgn_sum(const EvalArgs& A, int v, int e, int sol) {
  HGN r;
  r.h = r.g = 0.0;
  r.n = r.n0 = 0;
  for (int s = A.slab_off[e]; s < A.slab_off[e + 1]; s++) {
    const HGN x = A.hgn[((long long)v * A.n_slabs + s) * A.P + sol];
    r.h += x.h; r.g += x.g; r.n += x.n; r.n0 += x.n0;
  }
  return r;
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
    HGN r0 = hgn_sum(A, 0, e, sol);
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
        const HGN r1 = hgn_sum(A, 1, e, sol);
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
__global__ void k_own_records(const float* __restrict__ I, const unsigned char* __restrict__ band,
                              long long V, uint2* __restrict__ out) {
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < V;
       v += (long long)gridDim.x * blockDim.x)
    out[v] = make_uint2(__float_as_uint(I[v]), band ? (unsigned)band[v] : 0u);
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

cudaError_t launch_own_records(const float* I, const unsigned char* band, long long V, uint2* out,
                               cudaStream_t s) {
  k_own_records<<<2048, 256, 0, s>>>(I, band, V, out);
  return cudaGetLastError();
}

cudaError_t launch_band_mask(const float* dmap, int K, long long V, double r, unsigned char* band,
                             cudaStream_t s) {
  k_band_mask<<<2048, 256, 0, s>>>(dmap, K, V, r, band);
  return cudaGetLastError();
}

#include "morea_repair.cuh"
#include "morea_mix.cuh"

}  // namespace morea

#include "morea_sobol.cuh"

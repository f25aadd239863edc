// morea_export.cuh -- NEXT-4: rasterizer reuse (App. A.1,
// §5.4) on sm_100a, included by morea_kernels.cu (inside namespace morea).
//
//  * per-tet object counts for the elasticity factors c_delta ("We compute the
//    overlap that each object mask has with the tetrahedron ... one fraction per
//    object ... multiplied by pre-determined elasticity factors"), over the
//    exactly-once voxel centres each tet owns (E1, E2);
//  * the deformation vector field of one side (E3): T(q) - q in mm at every
//    owned voxel centre, from the exact int128 numerator rounded once to fp64 as
//    in the oracle, so the field is bit-identical to it.
// Both run the a4 rasterizer (raster()) with their own sample functors, one
// warp per tet, after k_setup has built the SideRecs (voxel-centre mode).
// (Included inside namespace morea.)
#pragma once

// E1: label = 1 + lowest set bit of the object byte below M, 0 = no object
__device__ __forceinline__ int voxel_label(unsigned m, int M) {
  const unsigned v = m & ((1u << M) - 1u);
  return v ? __ffs(v) : 0;
}

struct LabelSample {
  static constexpr bool kQuiet = false;
  __device__ __forceinline__ int quiet_off() const { return -1; }
  __device__ __forceinline__ unsigned quiet_hull(int) const { return 0xffff0000u; }
  __device__ __forceinline__ void count_quiet(int) {}
  __device__ __forceinline__ void quiet_row(int, int) {}
  const unsigned char* masks;
  int M;
  int* cnt;  // shared: M + 1 counters of this warp
  __device__ __forceinline__ void steps_done(int) {}
  __device__ __forceinline__ void flush_h() {}
  __device__ __forceinline__ void count_only(int) {}
  __device__ __forceinline__ void sample(const int4& ra, const float4&, int k, bool valid) {
    if (!valid) return;
    atomicAdd(&cnt[voxel_label(__ldg(&masks[ra.y + k]), M)], 1);
  }
};

__global__ void __launch_bounds__(kRasterThreads) k_label_counts(const EvalArgs A, int side,
                                                                 const unsigned char* __restrict__ masks,
                                                                 int M, long long* __restrict__ counts) {
  __shared__ WarpSmem smem[kWarpsPerBlock];
  __shared__ int cnt[kWarpsPerBlock][9];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tet = blockIdx.x * kWarpsPerBlock + warp;
  if (tet >= A.mesh.T) return;
  if (lane <= M) cnt[warp][lane] = 0;
  WarpSmem& S = smem[warp];
  load_rec(S, &A.geom[2 * (long long)tet + side], lane);
  if (S.R.flags & 1) {
    LabelSample f{masks, M, cnt[warp]};
    raster(S.R, A.vol.nx, A.vol.ny, 0, S, lane, f);
  }
  __syncwarp();
  if (lane <= M) counts[(long long)tet * (M + 1) + lane] = cnt[warp][lane];
}

// E3 pass 1: owner = lowest owning tet id (deterministic under folds)
struct MinOwnerSample {
  static constexpr bool kQuiet = false;
  __device__ __forceinline__ int quiet_off() const { return -1; }
  __device__ __forceinline__ unsigned quiet_hull(int) const { return 0xffff0000u; }
  __device__ __forceinline__ void count_quiet(int) {}
  __device__ __forceinline__ void quiet_row(int, int) {}
  int* owner;
  int tet;
  __device__ __forceinline__ void steps_done(int) {}
  __device__ __forceinline__ void flush_h() {}
  __device__ __forceinline__ void count_only(int) {}
  __device__ __forceinline__ void sample(const int4& ra, const float4&, int k, bool valid) {
    if (valid) atomicMin(&owner[ra.y + k], tet);
  }
};

// E3 pass 2: T(q) - q = sum_k e_k(q) U_k / (1024 |Delta|) (O4), exact numerator,
// one fp64 rounding (the oracle's operations), times the spacing, fp32
struct DvfSample {
  static constexpr bool kQuiet = false;
  __device__ __forceinline__ int quiet_off() const { return -1; }
  __device__ __forceinline__ unsigned quiet_hull(int) const { return 0xffff0000u; }
  __device__ __forceinline__ void count_quiet(int) {}
  __device__ __forceinline__ void quiet_row(int, int) {}
  const SideRec* R;  // shared
  const int* owner;
  int tet;
  double sp0, sp1, sp2;
  float* dvf;
  unsigned char* cov;
  __device__ __forceinline__ void steps_done(int) {}
  __device__ __forceinline__ void flush_h() {}
  __device__ __forceinline__ void count_only(int) {}
  __device__ __forceinline__ void sample(const int4& ra, const float4& rb, int k, bool valid) {
    if (!valid) return;
    const int lin = ra.y + k;
    if (__ldg(&owner[lin]) != tet) return;
    const int q[3] = {(int)rb.y + k, (int)rb.z, (int)rb.w};
    i64 e[4];
#pragma unroll
    for (int f = 0; f < 4; f++)
      e[f] = 1024 * (R->nrm[f][0] * q[0] + R->nrm[f][1] * q[1] + R->nrm[f][2] * q[2]) - R->cst[f];
    const double den = __dmul_rn((double)R->absdet, 1024.0);
    const double sp[3] = {sp0, sp1, sp2};
#pragma unroll
    for (int a = 0; a < 3; a++) {
      i128 n = 0;
#pragma unroll
      for (int f = 0; f < 4; f++) n += (i128)e[f] * (i128)R->U[f][a];
      const double u = __ddiv_rn((double)n, den);
      dvf[3LL * lin + a] = __double2float_rn(__dmul_rn(u, sp[a]));
    }
    cov[lin] = 1;
  }
};

__global__ void __launch_bounds__(kRasterThreads) k_min_owner(const EvalArgs A, int side, int* owner) {
  __shared__ WarpSmem smem[kWarpsPerBlock];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tet = blockIdx.x * kWarpsPerBlock + warp;
  if (tet >= A.mesh.T) return;
  WarpSmem& S = smem[warp];
  load_rec(S, &A.geom[2 * (long long)tet + side], lane);
  if (!(S.R.flags & 1)) return;
  MinOwnerSample f{owner, tet};
  raster(S.R, A.vol.nx, A.vol.ny, 0, S, lane, f);
}

__global__ void __launch_bounds__(kRasterThreads) k_dvf(const EvalArgs A, int side, const int* owner,
                                                        float* dvf, unsigned char* cov) {
  __shared__ WarpSmem smem[kWarpsPerBlock];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tet = blockIdx.x * kWarpsPerBlock + warp;
  if (tet >= A.mesh.T) return;
  WarpSmem& S = smem[warp];
  load_rec(S, &A.geom[2 * (long long)tet + side], lane);
  if (!(S.R.flags & 1)) return;
  DvfSample f{&S.R, owner, tet, A.vol.sp[0], A.vol.sp[1], A.vol.sp[2], dvf, cov};
  raster(S.R, A.vol.nx, A.vol.ny, 0, S, lane, f);
}

cudaError_t launch_label_counts(const EvalArgs& a, int side, const unsigned char* masks, int M,
                                long long* counts, cudaStream_t s) {
  cudaError_t e = launch_setup(a, s);
  if (e != cudaSuccess) return e;
  const int blocks = (a.mesh.T + kWarpsPerBlock - 1) / kWarpsPerBlock;
  k_label_counts<<<blocks, kRasterThreads, 0, s>>>(a, side, masks, M, counts);
  return cudaGetLastError();
}

cudaError_t launch_dvf(const EvalArgs& a, int side, int* owner, float* dvf, unsigned char* cov,
                       cudaStream_t s) {
  k_fill_int<<<1024, 256, 0, s>>>(owner, a.vol.V, 0x7fffffff);
  cudaError_t e = cudaMemsetAsync(dvf, 0, (size_t)a.vol.V * 3 * sizeof(float), s);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(cov, 0, (size_t)a.vol.V, s);
  if (e != cudaSuccess) return e;
  e = launch_setup(a, s);
  if (e != cudaSuccess) return e;
  const int blocks = (a.mesh.T + kWarpsPerBlock - 1) / kWarpsPerBlock;
  k_min_owner<<<blocks, kRasterThreads, 0, s>>>(a, side, owner);
  k_dvf<<<blocks, kRasterThreads, 0, s>>>(a, side, owner, dvf, cov);
  return cudaGetLastError();
}

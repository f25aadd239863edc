// Internal declarations shared by the host API (morea_api.cu) and the kernels
// (morea_kernels.cu).  Product code only; nothing here is shared with the
// independent CPU checker.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "morea.h"

// Debug builds (-DMOREA_DEBUG_CHECKS, tests/test_gpu_debug_checks.py) check index
// ranges and invariants on the device (assert traps); release builds compile the
// checks away.  (compute-sanitizer is closed on the GPU pool this was built on.)
#ifdef MOREA_DEBUG_CHECKS
#undef NDEBUG
#include <cassert>
#define MOREA_CHECK(c) assert(c)
#else
#define MOREA_CHECK(c) ((void)0)
#endif

namespace morea {

constexpr int kMaxPairs = 8;
constexpr int kTexPad = 1;  // edge-replicated border of the gather textures (voxels)
constexpr int kQLo = -256 * 1024;  // Q.10 window (O1)
constexpr int kQHi = 768 * 1024;
constexpr int kQuietRmin = 2, kQuietRmax = 15;  // radii of the empty-space row hulls (§4.10)
constexpr int kWarpsPerBlock = 2;  // k_owner_map / export blocks (one WarpSmem per warp)
constexpr int kRasterThreads = 32 * kWarpsPerBlock;

// Geometry of one (version, entry, solution, side) item, written by k_setup and
// read by k_raster.  384 bytes, 16-byte aligned.  The fp32 fields
// are roundings of exact (or fp64) values; each comes with an error bound so the
// rasterizer can detect when only the exact integer fields can decide.
struct __align__(16) SideRec {
  float4 face[4];             // (fa, fb, fc, thr): crossing x*(y,z) = fa + fb (y - lo_y) + fc (z - lo_z)
                              // and the bound on its fp32 error (voxels)
  int ftype[4];               // +-1: lower/upper bound face (n_x >< 0), 0: flat, +-2: exact search
  long long nrm[4][3];        // exact inward normals (|n| < 2^41)
  long long cst[4];           // e_k(q) = 1024 n_k . q - cst_k  (exact)
  float A[3][3];              // displacement gradient du_a / dq_b
  float d0[3];                // displacement at lo
  float eps[3];               // fp32 position filter bound per axis (0 = exact axis)
  int flags;                  // bit 0: rasterize; bit 1: every position of the bbox is inside
                              // [0, n-1) with margin (no clamp needed); bit 2: every face is a
                              // regular lower/upper face (fast row intervals); bit 3: every
                              // position is inside (-1, n) with margin (no clamp needed on the
                              // edge-padded gather textures); bits 8..15: empty-space radius R;
                              // bits 16..17: nl, regular items list their nl lower faces first
  float vy[4], vz[4];         // vertex y, z (voxel units, exact) for per-slice y ranges
  int lo[3], hi[3];           // lattice bbox clipped to the image
  int U[4][3];                // Q_other - Q_own per vertex
  long long absdet;           // |Delta|
};
static_assert(sizeof(SideRec) == 384, "SideRec layout");

// NEXT-1 (Sobol sampler, DESIGN.md §3 S1-S9): what k_sobol needs of one (version,
// entry, solution, side) item.  Written by k_setup into the item's SideRec slot.
struct __align__(16) SobolRec {
  int Q[4][3];              // sampled side, Q.10 (exact; the fp64 fallback recomputes from these)
  int Qo[4][3];             // other side
  float x0[3], D[3][3];     // sampled side: frac(X_0) and X_k - X_0 (k = 1..3), voxel units,
                            // fp32-exact; floor(X_0) in i0 (positions = i0 + x0 + sum l_k D_k)
  float x0o[3], Do[3][3];   // other side
  float i0[3], i0o[3];      // floor(X_0) per side (exact small integers as floats)
  unsigned mask[4];         // digital-shift masks (S3/S4)
  long long N;              // samples of this side (S6)
  float epsA, epsB;         // fast-path position error bound eps = epsA / s + epsB, s = sum -lg2 u
  int flags;                // bit 0: N > 0; bit 1: every vertex of both sides inside [0, n-1];
                            // bit 2: ... inside [-1 + 1/16, n - 1/16] (edge-padded textures)
  int pad;
};
static_assert(sizeof(SobolRec) == 256, "SobolRec layout");

// Per-tet scalar terms of one (version, entry, solution).
struct Scal {
  double m, sev;
  int folds, flags;  // flags bit 0: a vertex outside the Q.10 window
  int pad[2];
};
static_assert(sizeof(Scal) == 32, "Scal layout");

// Sample sums of one (version, entry, solution), both sides.
struct HGN {
  double h, g;
  long long n;   // samples (both sides)
  long long n0;  // samples of side 0 (coverage check)
};
static_assert(sizeof(HGN) == 32, "HGN layout");

struct Volumes {
  int nx, ny, nz;
  long long V;
  double sp[3];
  const float* I[2];
  const unsigned char* band[2];  // per voxel bit i = [D_i(q) < r]; nullptr when K == 0
  // per voxel (bits of I_side(q), band bits): one 8-byte load; one allocation,
  // own[1] = own[0] + V, so side s of voxel q is own[0][s V + q]
  const uint2* own[2];
  // empty space: per side, radius R in [kQuietRmin, kQuietRmax] and
  // image row (y, z), the first and last x whose quiet radius is < R ((nx, -1): none);
  // qhull[s] + (R - kQuietRmin) ny nz + z ny + y
  const short2* qhull[2];
  // per side and voxel v, the minimum quiet radius over the 4^3 block v - 1 .. v + 2
  // (clipped): the per-point empty-space test of the Sobol sampler
  const unsigned char* qcell[2];
  const float* dmap[2];          // K * V fp32 per side
  int K;
  double r, inv_r;
  float fnx2, fny2, fnz2;  // (n - 2) per axis as floats (constant-bank operands)
  const double* w;  // device: w[side * kMaxPairs + i] = |C_i| / |G_side|
  float wf[2][kMaxPairs];  // w / r (fp32), in the parameter space
  const float* wfd;        // the same, device memory [side * kMaxPairs + i] (runtime-indexed)
  float rf, rlo;           // r = rf + rlo (fp32 head and tail)
  // texture-gather path (0 when the layout exceeds the gather limits): volumes as
  // tall 2D textures with a one-voxel edge-replicated border, voxel (x, y, z) of
  // volume j -> texel (x + 1 + j (nx + 2), y + 1 + (ny + 2)(z + 1)) for x in
  // [-1, nx] etc. (indices clamped into the volume), gathered 2x2 per slice (tld4).
  // texI: volumes I_s, I_t; texM: the 2K maps, side s pair i at j = s K + i.
  // The border makes the O5 clamp implicit for positions in (-1, n): both
  // corners of a footprint straddling the border carry the border value.
  unsigned long long texI;
  unsigned long long texM;
  // gather coordinates of lower corner (ix, iy, iz) of volume j:
  //   u = ix + uoff0 + j fnxp,  v = fmaf(iz, fnyp, iy) + voff,  next slice v + fnyp
  // TEX: fnxp = nx + 2, fnyp = ny + 2, uoff0 = 2, voff = ny + 4 (padded layout);
  // plain loads: fnxp = nx, fnyp = ny, uoff0 = 1, voff = 1 (u - 1, v - 1 = index)
  float fnxp, fnyp, uoff0, voff;
  float uoffI[2];  // gather x offset of corner i0 of I_j: uoff0 + j fnxp
  int use_tex;
  // Sobol sampler (NEXT-1): per side and voxel v, OR of the band bits of v + {0,1}^3
  // (clamped): the pairs whose interpolated distance can be < r in v's cell
  const unsigned char* dil[2];
};

struct MeshDev {
  int N, T;
  const float* base;  // N*3
  const int4* tets;   // T
  const float* cdelta;
  const signed char* ref;
  int spoke_mode;
};

// One evaluation launch sequence: k_setup -> k_raster -> k_reduce.
// Item index space: (version, canonical entry, solution); version 0 = the new
// (evaluated) geometry, version 1 = the base geometry of a partial evaluation.
struct EvalArgs {
  Volumes vol;
  MeshDev mesh;
  int P;
  const float* offsets;      // P*N*6
  int n_entries;
  const int* canon_tet;      // canonical entry -> tet (nullptr: identity, full evaluation)
  const int4* canon_slots;   // canonical entry -> per vertex slot into new_vals, or -1
  const int* sched;          // queue position -> canonical entry (large tets first)
  const int* group_off;      // G + 1 offsets of the groups' canonical entries (k_reduce)
  const float* new_vals;     // P*S_total*6
  int S_total;
  int partial;
  int n_setup_versions;      // 1 (full) or 2 (partial)
  int n_raster_versions;     // 1, or 2 when a partial evaluation recomputes the base
  SideRec* geom;             // voxel-centre mode: [version][entry][sol][side]
  SobolRec* sgeom;           // Sobol mode: [version][entry][sol][side]
  Scal* scal;                // [version][entry][sol]
  HGN* hgn;                  // [version][entry][sol]
  long long expect[2];       // per-side sample count of the base mesh (coverage check), -1: off
  int sampler;               // 0: exactly-once voxel centres (k_raster), 1: Sobol points (k_sobol)
  double rate;               // Sobol samples per voxel of tet volume
  const unsigned* sobol_v;   // [4][32] Sobol direction numbers (device)
  int sobol_force_exact;     // test hook (env MOREA_SOBOL_FORCE_EXACT): every sample takes the fp64 path
  unsigned long long* counter;  // work queue head (zeroed before launch); debug builds: counter[1] =
                                // items processed, counter[2] = blocks finished (exactly-once check)
  unsigned long long* stats;    // [samples, band entries, items]
  float* dump_h;                // test hook morea_sample_map: per-voxel h and fg of side dump_side
  unsigned char* dump_fg;
  int dump_side;
};

// launches (morea_kernels.cu)
cudaError_t launch_validate_volume(const float* I, long long V, int* bad, cudaStream_t s);
cudaError_t launch_distance_maps(const float* pts, const long long* off, int K, int nx, int ny,
                                 int nz, const double sp[3], float* dmap, cudaStream_t s);
cudaError_t launch_band_mask(const float* dmap, int K, long long V, double r, unsigned char* band,
                             cudaStream_t s);
cudaError_t launch_pad_volume(const float* src, int nx, int ny, int nz, int pad, float* dst, cudaStream_t s);
cudaError_t launch_own_records(const float* I, const unsigned char* band, long long V,
                               uint2* out, cudaStream_t s);
cudaError_t launch_quiet_cells(const float* I, const unsigned char* band, const unsigned char* zr, int nx, int ny,
                               int nz, unsigned char* tmp0, unsigned char* tmp1, unsigned char* qcell, cudaStream_t s);
cudaError_t launch_quiet_hull(const float* I, const unsigned char* band, const unsigned char* zr, int nx, int ny,
                              int nz, short2* hull, cudaStream_t s);
cudaError_t launch_zero_radius(const float* I, int nx, int ny, int nz, unsigned char* zr, unsigned char* m0,
                               unsigned char* m1, cudaStream_t s);
cudaError_t launch_setup(const EvalArgs& a, cudaStream_t s);
cudaError_t launch_raster(const EvalArgs& a, int grid, cudaStream_t s);
int raster_blocks_per_sm(bool tex);
cudaError_t setup_prepare();  // k_setup's dynamic shared-memory opt-in (current device)
int raster_block_warps();
cudaError_t launch_sobol(const EvalArgs& a, int grid, cudaStream_t s);
int sobol_blocks_per_sm(bool tex);
int sobol_block_warps();
cudaError_t launch_repair(const MeshDev& m, const double sp[3], int P, long long sol_base, float* offsets,
                          const unsigned char* fixed, const int* inc_off, const int* inc,
                          unsigned long long seed, int* moved, int* aborted, cudaStream_t s);
cudaError_t launch_label_counts(const EvalArgs& a, int side, const unsigned char* masks, int M,
                                long long* counts, cudaStream_t s);
cudaError_t launch_dvf(const EvalArgs& a, int side, int* owner, float* dvf, unsigned char* cov,
                       cudaStream_t s);
// NEXT-3 sampling arguments (morea_mix.cuh)
struct MixArgs {
  int P, G, N, T, S_total, n_entries;
  long long sol_base;
  const float* offsets;        // P*N*6 (parent state)
  float* new_vals;             // P*S_total*6 (sampled)
  const int* grp_off;          // G+1 (device)
  const int* changed;          // S_total (device)
  const long long* model_off;  // G x 2: offsets of mu_g and L_g inside one cluster's block
  long long mu_stride, L_stride;  // doubles per cluster
  const int* cluster;          // P
  const double* mu;
  const double* L;
  const unsigned char* fixed;  // N*3 or nullptr
  unsigned long long seed;
  long long gen;
};
cudaError_t launch_mix_sample(const MixArgs& a, cudaStream_t s);
cudaError_t launch_mix_accept(int P, int G, int T, const morea_acc* base, const morea_acc* pacc, morea_acc* acc,
                              double* obj, const double* archive, int A_n, double steer_max,
                              unsigned char* accepted, cudaStream_t s);
cudaError_t launch_mix_commit(int P, int G, int N, int T, int S_total, int n_entries,
                              const unsigned char* accepted, const int* grp_off, const int* changed,
                              const int* group_off, const int* canon_tet, const float* new_vals,
                              const double* dep_cache, float* offsets, double* tet_cache, cudaStream_t s);
cudaError_t launch_dilate_band(const unsigned char* band, int nx, int ny, int nz, unsigned char* dil,
                               cudaStream_t s);
cudaError_t launch_reduce(const EvalArgs& a, int G, const int* group_off, const void* base_acc,
                          const double* cache_in, double* cache_out, const int* changed,
                          const int* grp_off, double* obj, void* acc, cudaStream_t s);
cudaError_t launch_check_folds(const MeshDev& m, const double sp[3], int P, const float* offsets,
                               int* count, double* sev, unsigned char* flags, cudaStream_t s);
cudaError_t launch_owner_map(const EvalArgs& a, int side, int* owner, cudaStream_t s);
cudaError_t launch_fill(float* h, unsigned char* fg, long long V, cudaStream_t s);

}  // namespace morea

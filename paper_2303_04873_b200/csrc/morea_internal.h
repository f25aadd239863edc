// Internal declarations shared by the host API (morea_api.cu) and the kernels
// (morea_kernels.cu).  Product code only -- nothing here is shared with the
// oracle under oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace morea {

constexpr int kMaxPairs = 8;
constexpr int kQLo = -256 * 1024;  // Q.10 window (O1)
constexpr int kQHi = 768 * 1024;
constexpr int kWarpsPerBlock = 8;
constexpr int kEvalThreads = 32 * kWarpsPerBlock;

// Per (solution, entry) record written by the evaluation kernel.
struct Rec {
  double h, g, m, sev;
  long long n;
  int folds, flags;  // flags bit 0: a vertex outside the window (domain)
};
static_assert(sizeof(Rec) == 48, "Rec layout");

struct Volumes {
  int nx, ny, nz;
  long long V;
  double sp[3];
  const float* I[2];
  const unsigned char* band[2];  // per voxel bit i = [D_i(q) < r]; nullptr when K == 0
  const float* dmap[2];          // K * V fp32 per side
  int K;
  double r;
  const double* w;  // device: w[side * kMaxPairs + i] = |C_i| / |G_side|
};

struct MeshDev {
  int N, T;
  const float* base;  // N*3
  const int4* tets;   // T
  const float* cdelta;
  const signed char* ref;
  int spoke_mode;
};

struct EvalArgs {
  Volumes vol;
  MeshDev mesh;
  int P;
  const float* offsets;  // P*N*6
  int n_entries;
  const int* entry_tet;      // schedule order (large tets first)
  const int* entry_out;      // canonical output index of the entry
  const int4* entry_slots;   // partial: per vertex slot into new_vals' S dim, or -1
  const float* new_vals;     // P*S_total*6
  int S_total;
  int partial;
  const double* cache_in;    // partial: P*T*4 old {h,g,n,m} or nullptr
  double* cache_out;         // full: P*T*4 by tet id; partial: P*n_out*4 by out index
  Rec* rec;                  // P*n_out
  int n_out;
  unsigned long long* counter;  // work queue head (zeroed before launch)
  unsigned long long* stats;    // [samples, band entries, items]
};

// launches (morea_kernels.cu)
cudaError_t launch_validate_volume(const float* I, long long V, int* bad, cudaStream_t s);
cudaError_t launch_distance_maps(const float* pts, const long long* off, int K, int nx, int ny,
                                 int nz, const double sp[3], float* dmap, cudaStream_t s);
cudaError_t launch_band_mask(const float* dmap, int K, long long V, double r, unsigned char* band,
                             cudaStream_t s);
cudaError_t launch_eval(const EvalArgs& a, int grid, cudaStream_t s);
int eval_blocks_per_sm();
cudaError_t launch_reduce(int P, int G, int n_out, const int* group_off, const Rec* rec,
                          const void* base_acc, int partial, int T, int N, const float* base,
                          const float* offsets, const int* changed, const int* grp_off,
                          const float* new_vals, int S_total, double* obj, void* acc,
                          cudaStream_t s);
cudaError_t launch_check_folds(const MeshDev& m, const double sp[3], int P, const float* offsets,
                               int* count, double* sev, unsigned char* flags, cudaStream_t s);
cudaError_t launch_owner_map(const Volumes& v, const MeshDev& m, const float* offsets_one,
                             int side, int* owner, cudaStream_t s);

}  // namespace morea

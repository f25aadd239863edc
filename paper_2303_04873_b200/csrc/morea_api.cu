// morea_api.cu -- host side of the C-ABI declared in include/morea.h.
//
// Validation, Q.10 canonicalisation of the base mesh and reference signs
// (App. A.4), incidence CSR and dependent-tet plans for partial
// evaluation (§4.2.1), host/device pointer staging, stream handling
// and kernel launches.  No arithmetic of the objectives happens here: every
// step of an evaluation runs in morea_kernels.cu.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <utility>
#include <vector>

#include "morea.h"
#include "morea_internal.h"

using namespace morea;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

// Page-locked host staging (uploads without a stream synchronisation).
struct PinnedBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    release();
    size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMallocHost(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
  ~PinnedBuf() { release(); }
};

// The static structure of one evaluation request (O10): canonical entries
// (dependent tets of each group, tets ascending within a group), their changed
// vertex slots and the (solution-independent) queue order.  Built on the host
// once per distinct FOS request, uploaded through
// pinned memory (no synchronisation), and kept in a small LRU cache.
struct Plan {
  std::vector<int32_t> key_off, key_pts;
  unsigned long long hash = 0, last_use = 0;
  int G = 0, S = 0, n_entries = 0;
  bool disjoint = true;  // dependent-tet sets pairwise disjoint (a colour class)
  std::vector<int32_t> dep_tets, dep_off;
  DevBuf dev;      // all device arrays below, one allocation
  PinnedBuf host;  // their staged copy (kept alive with the plan: the upload is async)
  const int* canon_tet = nullptr;  // nullptr: identity (the full plan)
  const int4* canon_slots = nullptr;
  const int* sched = nullptr;       // entries, largest tets first (k_setup, k_sobol)
  const int* group_off = nullptr;   // G + 1 offsets into the entries
  const int* grp_off = nullptr;     // G + 1 offsets into changed
  const int* changed = nullptr;     // S changed point ids
};
constexpr int kPlanCache = 64;  // distinct FOS requests kept (one per colour class and size)

}  // namespace

struct morea_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int n_sm = 148, blocks_per_sm = 1, blocks_per_sm_tex = 1;
  // images
  bool have_images = false;
  int nx = 0, ny = 0, nz = 0, K = 0;
  long long V = 0;
  double sp[3] = {1, 1, 1};
  double r = 0;
  double w[2][kMaxPairs] = {};
  DevBuf I[2], band[2], dmap[2], wts, own, qhull, qcell;
  // Sobol sampler (NEXT-1): mode, rate, dilated band masks (2 V bytes), direction numbers
  int sampler = MOREA_SAMPLER_VOXEL;
  double rate = 1.0;
  DevBuf dil, sobolv;
  // fold repair (NEXT-2): device incidence CSR, staging
  DevBuf d_inc_off, d_inc, st_fixed, st_rep;
  // rasterizer exports (NEXT-4)
  DevBuf st_masks, st_counts, st_dvf, st_cov, scratch_owner, zero_off;
  // optimal mixing (NEXT-3)
  DevBuf mx_off, mx_acc, mx_obj, mx_cache, mx_nv, mx_pobj, mx_pacc, mx_dep, mx_base, mx_accepted, mx_cluster,
      mx_mu, mx_L, mx_arch, mx_moff, mx_fixed;
  int blocks_per_sm_sobol = 1, blocks_per_sm_sobol_tex = 1;
  // texture-gather copies (tall 2D arrays) of I_s, I_t and the maps
  bool use_tex = false;
  cudaArray_t arrI = nullptr, arrM = nullptr;
  cudaTextureObject_t texI = 0, texM = 0;
  // mesh
  bool have_mesh = false;
  int N = 0, T = 0, spoke_mode = 0;
  DevBuf base, tets, cdelta, ref;
  std::vector<float> h_base;
  std::vector<int32_t> h_tets, inc_off, inc;
  std::vector<double> tet_size;
  long long expect[2] = {-1, -1};  // base-mesh sample counts per side (coverage check)
  // scratch
  DevBuf geom, sgeom, scal, hgn, counter, stats;
  DevBuf st_off, st_nv, st_cache_in, st_base_acc, st_obj, st_acc, st_cache_out, st_i32, st_f64,
      st_u8;
  std::unique_ptr<Plan> full;                 // all tets, one group (set_mesh)
  std::vector<std::unique_ptr<Plan>> plans;  // partial requests, LRU
  Plan* plan = nullptr;                      // the plan of the last partial / mixing call
  unsigned long long plan_clock = 0;
  // profiling
  bool prof = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs;
  long long prof_launches = 0;
  long long kernels = 0;  // every kernel launch of this context
  bool host_in = false;   // the current call staged a host input
};

namespace {

// NVTX range around an ABI call or a kernel launch (closed on every return path).
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};

int fail(morea_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return code;
}

#define CK(call)                                                                            \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      int code_ = (e_ == cudaErrorMemoryAllocation) ? MOREA_ENOMEM : MOREA_ECUDA;           \
      return fail(ctx, code_, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__,    \
                  __LINE__);                                                                \
    }                                                                                       \
  } while (0)

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Device view of an input: the pointer itself if it is device memory,
// otherwise an async copy into `st` (pageable sources are consumed before the
// call returns, so the caller may reuse them immediately).
// Host sources (pageable or pinned) are consumed before the call returns: a call
// that staged a pinned host input synchronises its stream before returning
// (finish_outputs), so the caller may refill the buffer at once.  Device inputs
// not 8-byte aligned are staged too (the kernels load offsets as float2).
cudaError_t in_dev(morea_ctx* ctx, const void* p, size_t bytes, DevBuf& st, const void** out) {
  if (!p || bytes == 0) {
    *out = p;
    return cudaSuccess;
  }
  const bool dev = is_device_ptr(p);
  if (dev && ((uintptr_t)p & 7u) == 0) {
    *out = p;
    return cudaSuccess;
  }
  cudaError_t e = st.ensure(bytes);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(st.p, p, bytes, dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ctx->stream);
  if (!dev) ctx->host_in = true;
  *out = st.p;
  return e;
}

struct OutView {
  void* user = nullptr;
  void* dev = nullptr;
  size_t bytes = 0;
  bool copy = false;
};

cudaError_t out_dev(void* p, size_t bytes, DevBuf& st, OutView& v) {
  v.user = p;
  v.bytes = bytes;
  v.copy = false;
  v.dev = p;
  if (!p || bytes == 0) return cudaSuccess;
  if (is_device_ptr(p)) return cudaSuccess;
  cudaError_t e = st.ensure(bytes);
  if (e != cudaSuccess) return e;
  v.dev = st.p;
  v.copy = true;
  return cudaSuccess;
}

// Copy staged outputs back and synchronise if any output was host memory.
cudaError_t finish_outputs(morea_ctx* ctx, OutView* v, int n) {
  bool any = ctx->host_in;
  ctx->host_in = false;
  for (int i = 0; i < n; i++) {
    if (!v[i].copy) continue;
    cudaError_t e = cudaMemcpyAsync(v[i].user, v[i].dev, v[i].bytes, cudaMemcpyDeviceToHost,
                                    ctx->stream);
    if (e != cudaSuccess) return e;
    any = true;
  }
  if (any) return cudaStreamSynchronize(ctx->stream);
  return cudaSuccess;
}

// Host copy of a small array that may live on either side.
template <class T>
cudaError_t to_host(morea_ctx* ctx, const T* p, size_t n, std::vector<T>& out) {
  out.resize(n);
  if (n == 0) return cudaSuccess;
  if (is_device_ptr(p)) {
    cudaError_t e = cudaMemcpyAsync(out.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost,
                                    ctx->stream);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(ctx->stream);
  }
  std::memcpy(out.data(), p, n * sizeof(T));
  return cudaSuccess;
}

// O1 on the host, used only for the base mesh (reference signs / validation):
// same fp64 operations as the device canon_q with a zero offset.
long long canon_host(float b) { return (long long)std::nearbyint(1024.0 * (double)b + 1024.0 * 0.0); }

__int128 det_host(const long long Q[4][3]) {
  __int128 a[3], b[3], c[3];
  for (int i = 0; i < 3; i++) {
    a[i] = Q[1][i] - Q[0][i];
    b[i] = Q[2][i] - Q[0][i];
    c[i] = Q[3][i] - Q[0][i];
  }
  return a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0]) +
         a[2] * (b[0] * c[1] - b[1] * c[0]);
}

Volumes volumes_of(const morea_ctx* c) {
  Volumes v;
  v.nx = c->nx; v.ny = c->ny; v.nz = c->nz; v.V = c->V;
  for (int a = 0; a < 3; a++) v.sp[a] = c->sp[a];
  for (int s = 0; s < 2; s++) {
    v.I[s] = c->I[s].as<float>();
    v.band[s] = c->K > 0 ? c->band[s].as<unsigned char>() : nullptr;
    v.dmap[s] = c->K > 0 ? c->dmap[s].as<float>() : nullptr;
    v.dil[s] = (c->K > 0 && c->dil.p) ? c->dil.as<unsigned char>() + (size_t)s * c->V : nullptr;
  }
  v.K = c->K;
  v.r = c->r;
  v.inv_r = c->r > 0 ? 1.0 / c->r : 0.0;
  v.fnx2 = (float)(c->nx - 2);
  v.fny2 = (float)(c->ny - 2);
  v.fnz2 = (float)(c->nz - 2);
  v.w = c->wts.as<double>();
  v.wfd = c->wts.p ? reinterpret_cast<const float*>(c->wts.as<double>() + 2 * kMaxPairs) : nullptr;
  for (int s = 0; s < 2; s++)
    for (int i = 0; i < kMaxPairs; i++) v.wf[s][i] = c->r > 0 ? (float)(c->w[s][i] / c->r) : 0.f;
  v.rf = (float)c->r;
  v.rlo = (float)(c->r - (double)v.rf);
  for (int s = 0; s < 2; s++) {
    v.qcell[s] = c->qcell.p ? c->qcell.as<unsigned char>() + (size_t)s * c->V : nullptr;
    v.qhull[s] = c->qhull.p ? c->qhull.as<short2>() + (size_t)s * (kQuietRmax - kQuietRmin + 1) * c->ny * c->nz
                            : nullptr;
  }
  v.own[0] = c->own.as<uint2>();
  v.own[1] = v.own[0] ? v.own[0] + c->V : nullptr;
  v.use_tex = c->use_tex ? 1 : 0;
  v.texI = c->texI;
  v.texM = c->texM;
  const int pad = c->use_tex ? kTexPad : 0;
  v.fnxp = (float)(c->nx + 2 * pad);
  v.fnyp = (float)(c->ny + 2 * pad);
  v.uoff0 = (float)(1 + pad);
  v.voff = (float)((c->ny + 2 * pad) * pad + pad + 1);
  for (int j = 0; j < 2; j++) v.uoffI[j] = v.uoff0 + (float)j * v.fnxp;
  return v;
}

MeshDev mesh_of(const morea_ctx* c) {
  MeshDev m;
  m.N = c->N; m.T = c->T;
  m.base = c->base.as<float>();
  m.tets = c->tets.as<int4>();
  m.cdelta = c->cdelta.as<float>();
  m.ref = c->ref.as<signed char>();
  m.spoke_mode = c->spoke_mode;
  return m;
}

constexpr long long kMixMaxDimHost = 192;  // = kMixMaxDim (morea_mix.cuh)

int raster_grid(morea_ctx* ctx, long long n_items) {
  long long g = (long long)ctx->n_sm * (ctx->use_tex ? ctx->blocks_per_sm_tex : ctx->blocks_per_sm);
  const int bw = raster_block_warps();
  long long need = (n_items + bw - 1) / bw;
  return (int)std::max<long long>(1, std::min(g, need));
}

void set_sampler_args(const morea_ctx* ctx, EvalArgs& a) {
  a.sampler = ctx->sampler;
  a.rate = ctx->rate;
  a.sobol_v = ctx->sobolv.as<unsigned>();
  const char* fe = std::getenv("MOREA_SOBOL_FORCE_EXACT");
  a.sobol_force_exact = (fe && fe[0] && fe[0] != '0') ? 1 : 0;
}

// Scratch for one evaluation: Scal per (version, entry, sol); SideRec (voxel
// centres) or SobolRec per rastered (version, entry, sol, side); HGN per
// rastered (version, entry, sol).
cudaError_t eval_scratch(morea_ctx* ctx, EvalArgs& a) {
  const size_t items = (size_t)a.n_entries * a.P;
  cudaError_t e = ctx->scal.ensure(std::max<size_t>(1, items * a.n_setup_versions) * sizeof(Scal));
  if (e != cudaSuccess) return e;
  e = ctx->hgn.ensure(std::max<size_t>(1, items * a.n_raster_versions) * sizeof(HGN));
  if (e != cudaSuccess) return e;
  a.scal = ctx->scal.as<Scal>();
  a.hgn = ctx->hgn.as<HGN>();
  if (a.sampler == MOREA_SAMPLER_SOBOL) {
    e = ctx->sgeom.ensure(std::max<size_t>(1, items * a.n_raster_versions * 2) * sizeof(SobolRec));
    if (e != cudaSuccess) return e;
    a.sgeom = ctx->sgeom.as<SobolRec>();
  } else {
    e = ctx->geom.ensure(std::max<size_t>(1, items * a.n_raster_versions * 2) * sizeof(SideRec));
    if (e != cudaSuccess) return e;
    a.geom = ctx->geom.as<SideRec>();
  }
  e = ctx->counter.ensure(3 * sizeof(unsigned long long));
  if (e != cudaSuccess) return e;
  a.counter = ctx->counter.as<unsigned long long>();
  a.stats = ctx->prof ? ctx->stats.as<unsigned long long>() : nullptr;
  return cudaSuccess;
}

// The plan's entries and queue order into the launch arguments.
void plan_args(const morea_ctx* ctx, const Plan& P, EvalArgs& a) {
  a.n_entries = P.n_entries;
  a.canon_tet = P.canon_tet;
  a.canon_slots = P.canon_slots;
  a.sched = P.sched;
  set_sampler_args(ctx, a);
}

// k_setup -> k_raster / k_sobol (the dominant kernel; bracketed by events when profiling).
cudaError_t run_eval(morea_ctx* ctx, EvalArgs& a) {
  cudaError_t e = eval_scratch(ctx, a);
  if (e != cudaSuccess) return e;
  {
    NvtxScope r("k_setup");
    e = launch_setup(a, ctx->stream);
  }
  ctx->kernels++;
  if (e != cudaSuccess) return e;
  const long long n_items = (long long)a.n_entries * a.P * a.n_raster_versions;
  if (n_items == 0) return cudaSuccess;
  e = cudaMemsetAsync(ctx->counter.p, 0, 3 * sizeof(unsigned long long), ctx->stream);
  if (e != cudaSuccess) return e;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ctx->prof) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, ctx->stream);
  }
  if (a.sampler == MOREA_SAMPLER_SOBOL) {
    NvtxScope r("k_sobol");
    const long long g = (long long)ctx->n_sm *
                        (ctx->use_tex ? ctx->blocks_per_sm_sobol_tex : ctx->blocks_per_sm_sobol);
    const long long need = (n_items + sobol_block_warps() - 1) / sobol_block_warps();
    e = launch_sobol(a, (int)std::max<long long>(1, std::min(g, need)), ctx->stream);
  } else {
    NvtxScope r("k_raster");
    e = launch_raster(a, raster_grid(ctx, n_items), ctx->stream);
  }
  ctx->kernels++;
  if (ctx->prof) {
    cudaEventRecord(e1, ctx->stream);
    ctx->evs.emplace_back(e0, e1);
    ctx->prof_launches++;
  }
  return e;
}

// Upload the plan's arrays in one allocation through pinned staging (no sync).
cudaError_t upload_plan(morea_ctx* ctx, Plan& P, const std::vector<int>& ct, const std::vector<int4>& cs,
                        const std::vector<int>& sched, const std::vector<int>& group_off,
                        const std::vector<int>& off, const std::vector<int>& pts, bool identity) {
  struct Seg { const void* src; size_t bytes; size_t at; };
  std::vector<Seg> segs;
  size_t tot = 0;
  auto add = [&](const void* src, size_t bytes) {
    tot = (tot + 15) & ~(size_t)15;
    segs.push_back({src, bytes, tot});
    tot += std::max<size_t>(bytes, 16);
    return segs.size() - 1;
  };
  const size_t i_ct = add(ct.data(), identity ? 0 : ct.size() * sizeof(int));
  const size_t i_cs = add(cs.data(), cs.size() * sizeof(int4));
  const size_t i_sc = add(sched.data(), sched.size() * sizeof(int));
  const size_t i_go = add(group_off.data(), group_off.size() * sizeof(int));
  const size_t i_of = add(off.data(), off.size() * sizeof(int));
  const size_t i_pt = add(pts.data(), pts.size() * sizeof(int));
  cudaError_t e = P.dev.ensure(tot);
  if (e != cudaSuccess) return e;
  e = P.host.ensure(tot);
  if (e != cudaSuccess) return e;
  for (const Seg& g : segs)
    if (g.bytes) std::memcpy((char*)P.host.p + g.at, g.src, g.bytes);
  e = cudaMemcpyAsync(P.dev.p, P.host.p, tot, cudaMemcpyHostToDevice, ctx->stream);
  if (e != cudaSuccess) return e;
  char* d = (char*)P.dev.p;
  P.canon_tet = identity ? nullptr : (const int*)(d + segs[i_ct].at);
  P.canon_slots = cs.empty() ? nullptr : (const int4*)(d + segs[i_cs].at);
  P.sched = (const int*)(d + segs[i_sc].at);
  P.group_off = (const int*)(d + segs[i_go].at);
  P.grp_off = (const int*)(d + segs[i_of].at);
  P.changed = (const int*)(d + segs[i_pt].at);
  return cudaSuccess;
}

unsigned long long plan_hash(const std::vector<int32_t>& off, const std::vector<int32_t>& pts) {
  unsigned long long h = 1469598103934665603ULL;
  auto mix = [&](int32_t v) {
    h ^= (unsigned)v;
    h *= 1099511628211ULL;
  };
  mix((int32_t)off.size());
  for (int32_t v : off) mix(v);
  for (int32_t v : pts) mix(v);
  return h;
}

// The dependent-tet plan of a partial request (host, O10), from the LRU cache
// or built and uploaded (asynchronously) on a miss.
int get_plan(morea_ctx* ctx, int G, const int32_t* grp_off_in, const int32_t* changed_in, Plan** out) {
  std::vector<int32_t> off, pts;
  CK(to_host(ctx, grp_off_in, (size_t)G + 1, off));
  if (off[0] != 0) return fail(ctx, MOREA_EINVAL, "grp_off[0] must be 0");
  for (int g = 0; g < G; g++)
    if (off[g + 1] < off[g]) return fail(ctx, MOREA_EINVAL, "grp_off must be non-decreasing");
  const int S = off[G];
  if (S > 0 && !changed_in) return fail(ctx, MOREA_EINVAL, "null changed_pts");
  CK(to_host(ctx, changed_in, (size_t)S, pts));
  const unsigned long long h = plan_hash(off, pts);
  for (auto& p : ctx->plans)
    if (p->hash == h && p->key_off == off && p->key_pts == pts) {
      p->last_use = ++ctx->plan_clock;
      *out = p.get();
      return MOREA_OK;
    }
  std::vector<int> stamp(ctx->N, -1), slot_of(ctx->N, -1), tstamp(ctx->T, -1), towner(ctx->T, -1);
  std::vector<int32_t> dep_tets, dep_off(1, 0);
  std::vector<int> ct;
  std::vector<int4> cs;
  bool disjoint = true;
  for (int g = 0; g < G; g++) {
    std::vector<int32_t> D;
    for (int i = off[g]; i < off[g + 1]; i++) {
      const int j = pts[i];
      if (j < 0 || j >= ctx->N) return fail(ctx, MOREA_EINVAL, "changed point %d out of range", j);
      if (stamp[j] == g) return fail(ctx, MOREA_EINVAL, "point %d twice in group %d", j, g);
      if (stamp[j] >= 0) disjoint = false;  // the point is in an earlier group too
      stamp[j] = g;
      slot_of[j] = i;
      for (int u = ctx->inc_off[j]; u < ctx->inc_off[j + 1]; u++) {
        const int t = ctx->inc[u];
        if (tstamp[t] != g) {
          tstamp[t] = g;
          D.push_back(t);
        }
      }
    }
    std::sort(D.begin(), D.end());
    for (int t : D) {
      if (towner[t] >= 0) disjoint = false;  // the tet depends on an earlier group too
      towner[t] = g;
      int s4[4];
      for (int k = 0; k < 4; k++) {
        const int j = ctx->h_tets[4 * t + k];
        s4[k] = stamp[j] == g ? slot_of[j] : -1;
      }
      ct.push_back(t);
      cs.push_back(make_int4(s4[0], s4[1], s4[2], s4[3]));
      dep_tets.push_back(t);
    }
    dep_off.push_back((int32_t)dep_tets.size());
  }
  const size_t ne = ct.size();
  std::vector<int> sched(ne);
  std::iota(sched.begin(), sched.end(), 0);
  std::stable_sort(sched.begin(), sched.end(),
                   [&](int a, int b) { return ctx->tet_size[ct[a]] > ctx->tet_size[ct[b]]; });
  std::unique_ptr<Plan> P(new Plan());
  P->key_off = off;
  P->key_pts = pts;
  P->hash = h;
  P->G = G;
  P->S = S;
  P->n_entries = (int)ne;
  P->disjoint = disjoint;
  P->dep_tets = dep_tets;
  P->dep_off = dep_off;
  CK(upload_plan(ctx, *P, ct, cs, sched, dep_off, off, pts, false));
  P->last_use = ++ctx->plan_clock;
  if ((int)ctx->plans.size() >= kPlanCache) {  // evict the least recently used
    size_t v = 0;
    for (size_t i = 1; i < ctx->plans.size(); i++)
      if (ctx->plans[i]->last_use < ctx->plans[v]->last_use) v = i;
    if (ctx->plan == ctx->plans[v].get()) ctx->plan = nullptr;
    CK(cudaStreamSynchronize(ctx->stream));  // its arrays may be in use by queued work
    ctx->plans.erase(ctx->plans.begin() + v);
  }
  *out = P.get();
  ctx->plans.push_back(std::move(P));
  return MOREA_OK;
}

// S1: direction numbers v_j[b] of the first four Sobol dimensions,
// row-major [4][32].  Dimension 0 is van der Corput (v = 2^(31-b)); dimensions
// 1..3 come from the primitive polynomials x + 1, x^2 + x + 1, x^3 + x + 1
// (degree s, inner coefficient bits a) with initial m = (1), (1, 3), (1, 3, 1)
// (Joe & Kuo), extended by the Bratley-Fox recurrence on the v's directly:
// v_b = v_{b-s} ^ (v_{b-s} >> s) ^ XOR_{k=1}^{s-1} a_k v_{b-k}.
std::vector<unsigned> sobol_directions() {
  struct Dim { int s; unsigned a; unsigned m[3]; };
  const Dim dims[3] = {{1, 0u, {1, 0, 0}}, {2, 1u, {1, 3, 0}}, {3, 1u, {1, 3, 1}}};
  std::vector<unsigned> v(4 * 32);
  for (int b = 0; b < 32; b++) v[b] = 1u << (31 - b);
  for (int d = 0; d < 3; d++) {
    unsigned* w = &v[32 * (d + 1)];
    const int s = dims[d].s;
    for (int b = 0; b < s; b++) w[b] = dims[d].m[b] << (31 - b);
    for (int b = s; b < 32; b++) {
      unsigned x = w[b - s] ^ (w[b - s] >> s);
      for (int k = 1; k < s; k++)
        if ((dims[d].a >> (s - 1 - k)) & 1u) x ^= w[b - k];
      w[b] = x;
    }
  }
  return v;
}

// dilated band masks for the Sobol sampler (built on demand)
cudaError_t ensure_dil(morea_ctx* ctx) {
  if (ctx->sampler != MOREA_SAMPLER_SOBOL || !ctx->have_images || ctx->K == 0 || ctx->dil.p)
    return cudaSuccess;
  cudaError_t e = ctx->dil.ensure(2 * (size_t)ctx->V);
  if (e != cudaSuccess) return e;
  for (int s = 0; s < 2; s++) {
    e = launch_dilate_band(ctx->band[s].as<unsigned char>(), ctx->nx, ctx->ny, ctx->nz,
                           ctx->dil.as<unsigned char>() + (size_t)s * ctx->V, ctx->stream);
    if (e != cudaSuccess) return e;
  }
  return cudaStreamSynchronize(ctx->stream);
}

void release_textures(morea_ctx* ctx) {
  if (ctx->texI) cudaDestroyTextureObject(ctx->texI);
  if (ctx->arrI) cudaFreeArray(ctx->arrI);
  if (ctx->texM) cudaDestroyTextureObject(ctx->texM);
  if (ctx->arrM) cudaFreeArray(ctx->arrM);
  ctx->texI = ctx->texM = 0;
  ctx->arrI = ctx->arrM = nullptr;
  ctx->use_tex = false;
}

// `count` float volumes (nx x ny x nz, x-fastest, device) as one 2D gather
// texture with a one-voxel edge-replicated border (Volumes::texI): volume j,
// voxel (x, y, z), x in [-1, nx] etc. -> texel (x + 1 + j (nx + 2),
// y + 1 + (ny + 2)(z + 1)).  Point sampling, clamp, unnormalised coordinates.
cudaError_t make_gather_texture(morea_ctx* ctx, const float* const* src, int count, cudaArray_t* arr,
                                cudaTextureObject_t* tex) {
  cudaChannelFormatDesc fd = cudaCreateChannelDesc<float>();
  const size_t wp = (size_t)ctx->nx + 2 * kTexPad, hp = ((size_t)ctx->ny + 2 * kTexPad) * ((size_t)ctx->nz + 2 * kTexPad);
#ifdef MOREA_TEX_ROUND
  const size_t W = (wp * count + MOREA_TEX_ROUND - 1) / MOREA_TEX_ROUND * MOREA_TEX_ROUND,
               H = (hp + MOREA_TEX_ROUND - 1) / MOREA_TEX_ROUND * MOREA_TEX_ROUND;
#else
  const size_t W = wp * count, H = hp;
#endif
  cudaError_t e = cudaMallocArray(arr, &fd, W, H, cudaArrayTextureGather);
  if (e != cudaSuccess) return e;
  float* padded = nullptr;
  e = cudaMallocAsync((void**)&padded, wp * hp * sizeof(float), ctx->stream);
  if (e != cudaSuccess) return e;
  for (int j = 0; j < count && e == cudaSuccess; j++) {
    e = launch_pad_volume(src[j], ctx->nx, ctx->ny, ctx->nz, kTexPad, padded, ctx->stream);
    if (e == cudaSuccess)
      e = cudaMemcpy2DToArrayAsync(*arr, (size_t)j * wp * sizeof(float), 0, padded, wp * sizeof(float),
                                   wp * sizeof(float), H, cudaMemcpyDeviceToDevice, ctx->stream);
  }
  const cudaError_t ef = cudaFreeAsync(padded, ctx->stream);
  if (e != cudaSuccess) return e;
  if (ef != cudaSuccess) return ef;
  cudaResourceDesc rd;
  std::memset(&rd, 0, sizeof(rd));
  rd.resType = cudaResourceTypeArray;
  rd.res.array.array = *arr;
  cudaTextureDesc td;
  std::memset(&td, 0, sizeof(td));
  td.addressMode[0] = td.addressMode[1] = cudaAddressModeClamp;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  return cudaCreateTextureObject(tex, &rd, &td, nullptr);
}

// Enable the texture-gather path when the tall 2D layout fits the gather limits.
cudaError_t build_textures(morea_ctx* ctx) {
  release_textures(ctx);
  const char* off = std::getenv("MOREA_NO_TEX");
  if (off && off[0] && off[0] != '0') return cudaSuccess;
  int gw = 0, gh = 0;
  cudaDeviceGetAttribute(&gw, cudaDevAttrMaxTexture2DGatherWidth, ctx->device);
  cudaDeviceGetAttribute(&gh, cudaDevAttrMaxTexture2DGatherHeight, ctx->device);
  if (((long long)ctx->nx + 2 * kTexPad) * 2 * std::max(ctx->K, 1) > gw ||
      ((long long)ctx->ny + 2 * kTexPad) * ((long long)ctx->nz + 2 * kTexPad) > gh)
    return cudaSuccess;
  const float* vols[2] = {ctx->I[0].as<float>(), ctx->I[1].as<float>()};
  cudaError_t e = make_gather_texture(ctx, vols, 2, &ctx->arrI, &ctx->texI);
  if (e != cudaSuccess) return e;
  if (ctx->K > 0) {
    std::vector<const float*> maps;
    for (int s = 0; s < 2; s++)
      for (int i = 0; i < ctx->K; i++) maps.push_back(ctx->dmap[s].as<float>() + (size_t)i * ctx->V);
    e = make_gather_texture(ctx, maps.data(), (int)maps.size(), &ctx->arrM, &ctx->texM);
    if (e != cudaSuccess) return e;
  }
  e = cudaStreamSynchronize(ctx->stream);
  if (e == cudaSuccess) ctx->use_tex = true;
  return e;
}

}  // namespace

extern "C" {

int morea_create(int cuda_device, void* cuda_stream, morea_ctx** out) {
  if (!out) return MOREA_EINVAL;
  *out = nullptr;
  morea_ctx* ctx = new morea_ctx();
  ctx->device = cuda_device;
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e != cudaSuccess) {
    delete ctx;
    return MOREA_ECUDA;
  }
  if (cuda_stream) {
    ctx->stream = (cudaStream_t)cuda_stream;
  } else {
    // blocking stream: implicitly ordered after work on the legacy default stream,
    // so inputs produced there (e.g. torch copies) are complete before our kernels run
    e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamDefault);
    if (e != cudaSuccess) {
      delete ctx;
      return MOREA_ECUDA;
    }
    ctx->own_stream = true;
  }
  cudaDeviceGetAttribute(&ctx->n_sm, cudaDevAttrMultiProcessorCount, cuda_device);
  if (setup_prepare() != cudaSuccess) {
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return MOREA_ECUDA;
  }
  ctx->blocks_per_sm = raster_blocks_per_sm(false);
  ctx->blocks_per_sm_tex = raster_blocks_per_sm(true);
  ctx->blocks_per_sm_sobol = sobol_blocks_per_sm(false);
  ctx->blocks_per_sm_sobol_tex = sobol_blocks_per_sm(true);
  {
    const std::vector<unsigned> v = sobol_directions();
    if (ctx->sobolv.ensure(v.size() * sizeof(unsigned)) != cudaSuccess ||
        cudaMemcpy(ctx->sobolv.p, v.data(), v.size() * sizeof(unsigned), cudaMemcpyHostToDevice) !=
            cudaSuccess) {
      delete ctx;
      return MOREA_ECUDA;
    }
  }
  if (ctx->stats.ensure(4 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemset(ctx->stats.p, 0, 4 * sizeof(unsigned long long)) != cudaSuccess) {
    delete ctx;
    return MOREA_ECUDA;
  }
  *out = ctx;
  return MOREA_OK;
}

void morea_destroy(morea_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  release_textures(ctx);
  for (auto& p : ctx->evs) {
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  DevBuf* bufs[] = {&ctx->I[0], &ctx->I[1], &ctx->band[0], &ctx->band[1], &ctx->dmap[0],
                    &ctx->dmap[1], &ctx->wts, &ctx->own, &ctx->qhull, &ctx->qcell, &ctx->dil, &ctx->sobolv, &ctx->d_inc_off, &ctx->d_inc, &ctx->st_fixed, &ctx->st_rep, &ctx->st_masks, &ctx->st_counts, &ctx->st_dvf, &ctx->st_cov,
                    &ctx->scratch_owner, &ctx->zero_off, &ctx->mx_off, &ctx->mx_acc,
                    &ctx->mx_obj, &ctx->mx_cache, &ctx->mx_nv, &ctx->mx_pobj, &ctx->mx_pacc, &ctx->mx_dep,
                    &ctx->mx_base, &ctx->mx_accepted, &ctx->mx_cluster, &ctx->mx_mu, &ctx->mx_L, &ctx->mx_arch,
                    &ctx->mx_moff, &ctx->mx_fixed, &ctx->base, &ctx->tets, &ctx->cdelta, &ctx->ref,
                    &ctx->geom, &ctx->sgeom, &ctx->scal, &ctx->hgn,
                    &ctx->counter, &ctx->stats, &ctx->st_off, &ctx->st_nv, &ctx->st_cache_in,
                    &ctx->st_base_acc, &ctx->st_obj, &ctx->st_acc, &ctx->st_cache_out,
                    &ctx->st_i32, &ctx->st_f64, &ctx->st_u8};
  for (DevBuf* b : bufs) b->release();
  for (auto& p : ctx->plans) p->dev.release();
  ctx->plans.clear();
  if (ctx->full) ctx->full->dev.release();
  ctx->full.reset();
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* morea_last_error(const morea_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void* morea_stream(const morea_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int morea_load_images(morea_ctx* ctx, int nx, int ny, int nz, const double spacing_mm[3],
                      const float* I_s, const float* I_t, int n_pairs, const int64_t* cs_off,
                      const float* cs_xyz, const int64_t* ct_off, const float* ct_xyz,
                      double r_mm) {
  NvtxScope nvtx_("morea_load_images");
  if (!ctx) return MOREA_EINVAL;
  CK(cudaSetDevice(ctx->device));
  if (nx < 2 || ny < 2 || nz < 2 || nx > 768 || ny > 768 || nz > 768)
    return fail(ctx, MOREA_EINVAL, "dims must be in [2, 768], got %d x %d x %d", nx, ny, nz);
  if (!spacing_mm || !I_s || !I_t) return fail(ctx, MOREA_EINVAL, "null spacing or volume");
  std::vector<double> sp;
  CK(to_host(ctx, spacing_mm, 3, sp));
  for (int a = 0; a < 3; a++)
    if (!(sp[a] > 0.0) || !std::isfinite(sp[a])) return fail(ctx, MOREA_EINVAL, "spacing must be > 0");
  if (n_pairs < 0 || n_pairs > kMaxPairs)
    return fail(ctx, MOREA_EINVAL, "n_pairs must be in [0, %d]", kMaxPairs);
  ctx->have_images = false;
  ctx->have_mesh = false;
  ctx->plans.clear();
  ctx->plan = nullptr;
  const long long V = (long long)nx * ny * nz;
  ctx->nx = nx; ctx->ny = ny; ctx->nz = nz; ctx->V = V;
  for (int a = 0; a < 3; a++) ctx->sp[a] = sp[a];
  const float* Iin[2] = {I_s, I_t};
  CK(ctx->st_i32.ensure(sizeof(int)));
  CK(cudaMemsetAsync(ctx->st_i32.p, 0, sizeof(int), ctx->stream));
  for (int s = 0; s < 2; s++) {
    CK(ctx->I[s].ensure(V * sizeof(float)));
    CK(cudaMemcpyAsync(ctx->I[s].p, Iin[s], V * sizeof(float), cudaMemcpyDefault, ctx->stream));
    CK(launch_validate_volume(ctx->I[s].as<float>(), V, ctx->st_i32.as<int>(), ctx->stream));
  }
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, ctx->st_i32.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (bad) return fail(ctx, MOREA_EINVAL, "intensities must be finite, and 0 or in [2^-40, inf)");
  // contours
  const int K = n_pairs;
  ctx->K = K;
  ctx->r = r_mm > 0.0 ? r_mm : 0.025 * (double)nx * sp[0];  // App. A.3
  const int64_t* offs[2] = {cs_off, ct_off};
  const float* xyz[2] = {cs_xyz, ct_xyz};
  std::memset(ctx->w, 0, sizeof(ctx->w));
  for (int s = 0; s < 2 && K > 0; s++) {
    std::vector<int64_t> off;
    if (!offs[s]) return fail(ctx, MOREA_EINVAL, "null contour offsets");
    CK(to_host(ctx, offs[s], (size_t)K + 1, off));
    if (off[0] != 0) return fail(ctx, MOREA_EINVAL, "contour offsets must start at 0");
    for (int i = 0; i < K; i++)
      if (off[i + 1] < off[i]) return fail(ctx, MOREA_EINVAL, "contour offsets must be non-decreasing");
    const int64_t M = off[K];
    if (M > 0 && !xyz[s]) return fail(ctx, MOREA_EINVAL, "null contour points");
    for (int i = 0; i < K; i++) ctx->w[s][i] = M > 0 ? (double)(off[i + 1] - off[i]) / (double)M : 0.0;
    DevBuf pts, doff;
    CK(pts.ensure(std::max<int64_t>(M, 1) * 3 * sizeof(float)));
    CK(doff.ensure((K + 1) * sizeof(long long)));
    if (M > 0) CK(cudaMemcpyAsync(pts.p, xyz[s], M * 3 * sizeof(float), cudaMemcpyDefault, ctx->stream));
    CK(cudaMemcpyAsync(doff.p, off.data(), (K + 1) * sizeof(long long), cudaMemcpyHostToDevice, ctx->stream));
    CK(ctx->dmap[s].ensure((size_t)K * V * sizeof(float)));
    CK(ctx->band[s].ensure(V));
    CK(launch_distance_maps(pts.as<float>(), doff.as<long long>(), K, nx, ny, nz, ctx->sp,
                            ctx->dmap[s].as<float>(), ctx->stream));
    CK(launch_band_mask(ctx->dmap[s].as<float>(), K, V, ctx->r, ctx->band[s].as<unsigned char>(),
                        ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    pts.release();
    doff.release();
  }
  // device weights: w (fp64, 2 x kMaxPairs) then w / r (fp32, 2 x kMaxPairs)
  CK(ctx->wts.ensure(sizeof(ctx->w) + 2 * kMaxPairs * sizeof(float)));
  CK(cudaMemcpyAsync(ctx->wts.p, ctx->w, sizeof(ctx->w), cudaMemcpyHostToDevice, ctx->stream));
  {
    std::vector<float> wf(2 * kMaxPairs);
    for (int s = 0; s < 2; s++)
      for (int i = 0; i < kMaxPairs; i++) wf[s * kMaxPairs + i] = ctx->r > 0 ? (float)(ctx->w[s][i] / ctx->r) : 0.f;
    CK(cudaMemcpy((char*)ctx->wts.p + sizeof(ctx->w), wf.data(), wf.size() * sizeof(float), cudaMemcpyHostToDevice));
  }
  CK(ctx->own.ensure(2 * V * sizeof(uint2)));
  {
    DevBuf zr, m0, m1;  // zero radius of the other volume (empty-space skipping)
    CK(zr.ensure(V));
    CK(m0.ensure(V));
    CK(m1.ensure(V));
    const size_t nh = (size_t)(kQuietRmax - kQuietRmin + 1) * ny * nz;
    CK(ctx->qhull.ensure(2 * nh * sizeof(short2)));
    CK(ctx->qcell.ensure(2 * V));
    for (int s = 0; s < 2; s++) {
      CK(launch_zero_radius(ctx->I[1 - s].as<float>(), nx, ny, nz, zr.as<unsigned char>(), m0.as<unsigned char>(),
                            m1.as<unsigned char>(), ctx->stream));
      CK(launch_own_records(ctx->I[s].as<float>(), K > 0 ? ctx->band[s].as<unsigned char>() : nullptr, V,
                            ctx->own.as<uint2>() + (size_t)s * V, ctx->stream));
      CK(launch_quiet_hull(ctx->I[s].as<float>(), K > 0 ? ctx->band[s].as<unsigned char>() : nullptr,
                           zr.as<unsigned char>(), nx, ny, nz, ctx->qhull.as<short2>() + (size_t)s * nh, ctx->stream));
      CK(launch_quiet_cells(ctx->I[s].as<float>(), K > 0 ? ctx->band[s].as<unsigned char>() : nullptr,
                            zr.as<unsigned char>(), nx, ny, nz, m0.as<unsigned char>(), m1.as<unsigned char>(),
                            ctx->qcell.as<unsigned char>() + (size_t)s * V, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  CK(build_textures(ctx));
  ctx->dil.release();
  ctx->have_images = true;
  CK(ensure_dil(ctx));
  return MOREA_OK;
}

int morea_set_mesh(morea_ctx* ctx, int n_points, const float* base_xyz, int n_tets,
                   const int32_t* tets, const float* c_delta, int spoke_mode) {
  NvtxScope nvtx_("morea_set_mesh");
  if (!ctx) return MOREA_EINVAL;
  CK(cudaSetDevice(ctx->device));
  if (!ctx->have_images) return fail(ctx, MOREA_ESTATE, "morea_load_images must come first");
  if (n_points < 4 || n_tets < 1 || !base_xyz || !tets)
    return fail(ctx, MOREA_EINVAL, "need >= 4 points and >= 1 tet");
  if (spoke_mode != MOREA_SPOKE_FACE_CENTROID && spoke_mode != MOREA_SPOKE_TET_CENTROID)
    return fail(ctx, MOREA_EINVAL, "bad spoke_mode");
  ctx->have_mesh = false;
  CK(cudaStreamSynchronize(ctx->stream));  // cached plans may be in use by queued work
  ctx->plans.clear();
  ctx->plan = nullptr;
  std::vector<float> b, cd;
  std::vector<int32_t> t;
  CK(to_host(ctx, base_xyz, (size_t)n_points * 3, b));
  CK(to_host(ctx, tets, (size_t)n_tets * 4, t));
  if (c_delta) {
    CK(to_host(ctx, c_delta, (size_t)n_tets, cd));
  } else {
    cd.assign(n_tets, 1.0f);
  }
  for (int i = 0; i < 4 * n_tets; i++)
    if (t[i] < 0 || t[i] >= n_points) return fail(ctx, MOREA_EINVAL, "tet index %d out of range", t[i]);
  for (int i = 0; i < n_tets; i++)
    if (!std::isfinite(cd[i])) return fail(ctx, MOREA_EINVAL, "c_delta must be finite");
  std::vector<long long> Q((size_t)n_points * 3);
  for (int j = 0; j < n_points; j++)
    for (int a = 0; a < 3; a++) {
      if (!std::isfinite(b[3 * j + a])) return fail(ctx, MOREA_EINVAL, "base point %d not finite", j);
      Q[3 * j + a] = canon_host(b[3 * j + a]);
      if (Q[3 * j + a] < kQLo || Q[3 * j + a] >= kQHi)
        return fail(ctx, MOREA_EDOMAIN, "base point %d outside the Q.10 window", j);
    }
  std::vector<signed char> ref(n_tets);
  std::vector<double> size(n_tets);
  for (int i = 0; i < n_tets; i++) {
    long long q[4][3];
    for (int k = 0; k < 4; k++)
      for (int a = 0; a < 3; a++) q[k][a] = Q[3 * t[4 * i + k] + a];
    __int128 d = det_host(q);
    if (d == 0) return fail(ctx, MOREA_EDOMAIN, "base tet %d has zero volume", i);
    ref[i] = d > 0 ? 1 : -1;  // reference signs, App. A.4
    size[i] = std::fabs((double)d);
  }
  // incidence CSR (tets incident to each point, ascending)
  std::vector<int32_t> inc_off(n_points + 1, 0), inc;
  for (int i = 0; i < n_tets; i++) {
    int v[4] = {t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3]};
    for (int k = 0; k < 4; k++) {
      bool dup = false;
      for (int l = 0; l < k; l++) dup = dup || v[l] == v[k];
      if (!dup) inc_off[v[k] + 1]++;
    }
  }
  for (int j = 0; j < n_points; j++) inc_off[j + 1] += inc_off[j];
  inc.resize(inc_off[n_points]);
  std::vector<int32_t> fill(inc_off.begin(), inc_off.end() - 1);
  for (int i = 0; i < n_tets; i++) {
    int v[4] = {t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3]};
    for (int k = 0; k < 4; k++) {
      bool dup = false;
      for (int l = 0; l < k; l++) dup = dup || v[l] == v[k];
      if (!dup) inc[fill[v[k]]++] = i;
    }
  }
  ctx->N = n_points;
  ctx->T = n_tets;
  ctx->spoke_mode = spoke_mode;
  ctx->h_base = b;
  ctx->h_tets = t;
  ctx->inc_off = inc_off;
  ctx->inc = inc;
  CK(ctx->d_inc_off.ensure(inc_off.size() * sizeof(int32_t)));
  CK(ctx->d_inc.ensure(std::max<size_t>(1, inc.size()) * sizeof(int32_t)));
  CK(cudaMemcpyAsync(ctx->d_inc_off.p, inc_off.data(), inc_off.size() * sizeof(int32_t),
                     cudaMemcpyHostToDevice, ctx->stream));
  if (!inc.empty())
    CK(cudaMemcpyAsync(ctx->d_inc.p, inc.data(), inc.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                       ctx->stream));
  ctx->tet_size = size;
  std::vector<int> order(n_tets), all(n_tets);
  std::iota(order.begin(), order.end(), 0);
  std::iota(all.begin(), all.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int c) { return size[a] > size[c]; });
  const std::vector<int> goff = {0, n_tets};
  CK(ctx->base.ensure(b.size() * sizeof(float)));
  CK(ctx->tets.ensure(t.size() * sizeof(int32_t)));
  CK(ctx->cdelta.ensure(cd.size() * sizeof(float)));
  CK(ctx->ref.ensure(ref.size()));
  CK(cudaMemcpyAsync(ctx->base.p, b.data(), b.size() * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->tets.p, t.data(), t.size() * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->cdelta.p, cd.data(), cd.size() * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->ref.p, ref.data(), ref.size(), cudaMemcpyHostToDevice, ctx->stream));
  // the full-evaluation plan: every tet, one group, identity entries
  ctx->full.reset(new Plan());
  ctx->full->G = 1;
  ctx->full->n_entries = n_tets;
  CK(upload_plan(ctx, *ctx->full, all, std::vector<int4>(), order, goff, std::vector<int>{0}, std::vector<int>(),
                 true));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->have_mesh = true;
  // coverage reference: per-side owned-sample counts of the base mesh (zero offsets)
  {
    ctx->expect[0] = ctx->expect[1] = -1;
    DevBuf zoff;
    CK(zoff.ensure((size_t)n_points * 6 * sizeof(float)));
    CK(cudaMemsetAsync(zoff.p, 0, (size_t)n_points * 6 * sizeof(float), ctx->stream));
    EvalArgs a;
    std::memset(&a, 0, sizeof(a));
    a.vol = volumes_of(ctx);
    a.mesh = mesh_of(ctx);
    a.P = 1;
    a.offsets = zoff.as<float>();
    plan_args(ctx, *ctx->full, a);
    a.sampler = MOREA_SAMPLER_VOXEL;  // the coverage reference is always voxel centres
    a.n_setup_versions = 1;
    a.n_raster_versions = 1;
    a.expect[0] = a.expect[1] = -1;
    CK(run_eval(ctx, a));
    std::vector<HGN> hg(n_tets);
    CK(cudaMemcpyAsync(hg.data(), ctx->hgn.p, hg.size() * sizeof(HGN), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    long long c0 = 0, c1 = 0;
    for (const HGN& x : hg) {
      c0 += x.n0;
      c1 += x.n - x.n0;
    }
    ctx->expect[0] = c0;
    ctx->expect[1] = c1;
    zoff.release();
    if (ctx->prof) {  // not part of any measured evaluation
      for (auto& p : ctx->evs) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
      ctx->evs.clear();
      ctx->prof_launches = 0;
    }
  }
  return MOREA_OK;
}

static int check_ready(morea_ctx* ctx) {
  if (!ctx) return MOREA_EINVAL;
  if (!ctx->have_images || !ctx->have_mesh)
    return fail(ctx, MOREA_ESTATE, "load images and set the mesh before evaluating");
  return MOREA_OK;
}

int morea_eval_full(morea_ctx* ctx, int pop, const float* offsets, double* obj, morea_acc* acc,
                    double* tet_cache) {
  int rc = check_ready(ctx);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  if (pop < 0 || (pop > 0 && !offsets)) return fail(ctx, MOREA_EINVAL, "bad pop / offsets");
  if (pop == 0) return MOREA_OK;
  NvtxScope nvtx_("morea_eval_full");
  const int N = ctx->N, T = ctx->T;
  const float* off = nullptr;
  ctx->host_in = false;
  CK(in_dev(ctx, offsets, (size_t)pop * N * 6 * sizeof(float), ctx->st_off, (const void**)&off));
  OutView ov[3];
  CK(out_dev(obj, (size_t)pop * 3 * sizeof(double), ctx->st_obj, ov[0]));
  CK(out_dev(acc, (size_t)pop * sizeof(morea_acc), ctx->st_acc, ov[1]));
  CK(out_dev(tet_cache, (size_t)pop * T * 4 * sizeof(double), ctx->st_cache_out, ov[2]));
  EvalArgs a;
  std::memset(&a, 0, sizeof(a));
  a.vol = volumes_of(ctx);
  a.mesh = mesh_of(ctx);
  a.P = pop;
  a.offsets = off;
  plan_args(ctx, *ctx->full, a);
  a.partial = 0;
  a.n_setup_versions = 1;
  a.n_raster_versions = 1;
  a.expect[0] = ctx->sampler == MOREA_SAMPLER_VOXEL ? ctx->expect[0] : -1;
  a.expect[1] = ctx->sampler == MOREA_SAMPLER_VOXEL ? ctx->expect[1] : -1;
  CK(run_eval(ctx, a));
  CK(launch_reduce(a, 1, ctx->full->group_off, nullptr, nullptr, (double*)ov[2].dev, nullptr, nullptr,
                   (double*)ov[0].dev, ov[1].dev, ctx->stream));
  ctx->kernels++;
  CK(finish_outputs(ctx, ov, 3));
  return MOREA_OK;
}

// a8 on device buffers: the plan P, base offsets/acc, new values, optional
// cache; outputs per (solution, group) and the dependent-tet cache rows
static cudaError_t partial_core(morea_ctx* ctx, const Plan& P, int pop, int G, const float* off,
                                const morea_acc* bacc, const float* nv, const double* cin, double* obj,
                                morea_acc* acc, double* dep_out) {
  EvalArgs a;
  std::memset(&a, 0, sizeof(a));
  a.vol = volumes_of(ctx);
  a.mesh = mesh_of(ctx);
  a.P = pop;
  a.offsets = off;
  plan_args(ctx, P, a);
  a.new_vals = nv;
  a.S_total = P.S;
  a.partial = 1;
  a.n_setup_versions = 2;
  a.n_raster_versions = cin ? 1 : 2;
  a.expect[0] = a.expect[1] = -1;
  cudaError_t e = run_eval(ctx, a);
  if (e != cudaSuccess) return e;
  e = launch_reduce(a, G, P.group_off, bacc, cin, dep_out, P.changed, P.grp_off, obj, acc, ctx->stream);
  ctx->kernels++;
  return e;
}

int morea_prepare_partial(morea_ctx* ctx, int n_groups, const int32_t* grp_off, const int32_t* changed_pts) {
  NvtxScope nvtx_("morea_prepare_partial");
  int rc = check_ready(ctx);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  if (n_groups < 0 || !grp_off) return fail(ctx, MOREA_EINVAL, "bad groups");
  Plan* P = nullptr;
  rc = get_plan(ctx, n_groups, grp_off, changed_pts, &P);
  if (rc) return rc;
  ctx->plan = P;
  return MOREA_OK;
}

int morea_eval_partial(morea_ctx* ctx, int pop, const float* base_offsets,
                       const morea_acc* base_acc, int n_groups, const int32_t* grp_off,
                       const int32_t* changed_pts, const float* new_vals, const double* tet_cache,
                       double* obj, morea_acc* acc, double* dep_cache_out) {
  int rc = check_ready(ctx);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  if (pop < 0 || n_groups < 0 || !grp_off) return fail(ctx, MOREA_EINVAL, "bad pop / groups");
  if (pop > 0 && (!base_offsets || !base_acc)) return fail(ctx, MOREA_EINVAL, "null base inputs");
  NvtxScope nvtx_("morea_eval_partial");
  Plan* Pp = nullptr;
  rc = get_plan(ctx, n_groups, grp_off, changed_pts, &Pp);
  if (rc) return rc;
  ctx->plan = Pp;
  const Plan& P = *Pp;
  if (pop == 0 || n_groups == 0) return MOREA_OK;
  if (P.S > 0 && !new_vals) return fail(ctx, MOREA_EINVAL, "null new_vals");
  const int N = ctx->N, T = ctx->T, G = n_groups;
  const float *off = nullptr, *nv = nullptr;
  const double* cin = nullptr;
  const morea_acc* bacc = nullptr;
  ctx->host_in = false;
  CK(in_dev(ctx, base_offsets, (size_t)pop * N * 6 * sizeof(float), ctx->st_off, (const void**)&off));
  CK(in_dev(ctx, new_vals, (size_t)pop * P.S * 6 * sizeof(float), ctx->st_nv, (const void**)&nv));
  CK(in_dev(ctx, tet_cache, (size_t)pop * T * 4 * sizeof(double), ctx->st_cache_in, (const void**)&cin));
  CK(in_dev(ctx, base_acc, (size_t)pop * sizeof(morea_acc), ctx->st_base_acc, (const void**)&bacc));
  OutView ov[3];
  CK(out_dev(obj, (size_t)pop * G * 3 * sizeof(double), ctx->st_obj, ov[0]));
  CK(out_dev(acc, (size_t)pop * G * sizeof(morea_acc), ctx->st_acc, ov[1]));
  CK(out_dev(dep_cache_out, (size_t)pop * P.n_entries * 4 * sizeof(double), ctx->st_cache_out, ov[2]));
  CK(partial_core(ctx, P, pop, G, off, bacc, nv, cin, (double*)ov[0].dev, (morea_acc*)ov[1].dev,
                  (double*)ov[2].dev));
  CK(finish_outputs(ctx, ov, 3));
  return MOREA_OK;
}

int morea_set_sampler(morea_ctx* ctx, int mode, double rate) {
  NvtxScope nvtx_("morea_set_sampler");
  if (!ctx) return MOREA_EINVAL;
  if (mode != MOREA_SAMPLER_VOXEL && mode != MOREA_SAMPLER_SOBOL)
    return fail(ctx, MOREA_EINVAL, "unknown sampler mode %d", mode);
  if (!(rate > 0.0 && rate <= 8.0)) return fail(ctx, MOREA_EINVAL, "rate must be in (0, 8] (32-bit per-tet counts)");
  CK(cudaSetDevice(ctx->device));
  ctx->sampler = mode;
  ctx->rate = rate;
  CK(ensure_dil(ctx));
  return MOREA_OK;
}

int morea_repair(morea_ctx* ctx, int pop, float* offsets, const uint8_t* fixed, uint64_t seed,
                 int64_t sol_base, int32_t* moved, int32_t* aborted) {
  NvtxScope nvtx_("morea_repair");
  int rc = check_ready(ctx);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  if (pop < 0 || (pop > 0 && !offsets) || sol_base < 0) return fail(ctx, MOREA_EINVAL, "bad pop / offsets");
  if (pop == 0) return MOREA_OK;
  const size_t bytes = (size_t)pop * ctx->N * 6 * sizeof(float);
  OutView ov[3];
  CK(out_dev(offsets, bytes, ctx->st_rep, ov[0]));
  if (ov[0].copy)  // in/out: bring the host offsets over first
    CK(cudaMemcpyAsync(ov[0].dev, offsets, bytes, cudaMemcpyHostToDevice, ctx->stream));
  const unsigned char* fx = nullptr;
  CK(in_dev(ctx, fixed, (size_t)ctx->N * 3, ctx->st_fixed, (const void**)&fx));
  CK(out_dev(moved, (size_t)pop * sizeof(int32_t), ctx->st_i32, ov[1]));
  CK(out_dev(aborted, (size_t)pop * sizeof(int32_t), ctx->st_u8, ov[2]));
  CK(launch_repair(mesh_of(ctx), ctx->sp, pop, sol_base, (float*)ov[0].dev, fx, ctx->d_inc_off.as<int>(),
                   ctx->d_inc.as<int>(), seed, (int*)ov[1].dev, (int*)ov[2].dev, ctx->stream));
  ctx->kernels++;
  CK(finish_outputs(ctx, ov, 3));
  return MOREA_OK;
}

// one-solution geometry (voxel-centre mode) for the rasterizer exports
static int export_args(morea_ctx* ctx, const float* offsets_one, EvalArgs& a) {
  const float* off = nullptr;
  if (offsets_one) {
    CK(in_dev(ctx, offsets_one, (size_t)ctx->N * 6 * sizeof(float), ctx->st_off, (const void**)&off));
  } else {
    CK(ctx->zero_off.ensure((size_t)ctx->N * 6 * sizeof(float)));
    CK(cudaMemsetAsync(ctx->zero_off.p, 0, (size_t)ctx->N * 6 * sizeof(float), ctx->stream));
    off = ctx->zero_off.as<float>();
  }
  std::memset(&a, 0, sizeof(a));
  a.vol = volumes_of(ctx);
  a.mesh = mesh_of(ctx);
  a.P = 1;
  a.offsets = off;
  plan_args(ctx, *ctx->full, a);
  a.sampler = MOREA_SAMPLER_VOXEL;  // the exports always use the voxel-centre sample set
  a.n_setup_versions = 1;
  a.n_raster_versions = 1;
  a.expect[0] = a.expect[1] = -1;
  CK(eval_scratch(ctx, a));
  return MOREA_OK;
}

int morea_label_counts(morea_ctx* ctx, const float* offsets_one, int side, const uint8_t* masks, int M,
                       int64_t* counts) {
  NvtxScope nvtx_("morea_label_counts");
  int rc = check_ready(ctx);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  if ((side != 0 && side != 1) || M < 0 || M > 8 || !masks || !counts)
    return fail(ctx, MOREA_EINVAL, "bad side / M / buffers");
  EvalArgs a;
  rc = export_args(ctx, offsets_one, a);
  if (rc) return rc;
  const unsigned char* m = nullptr;
  CK(in_dev(ctx, masks, (size_t)ctx->V, ctx->st_masks, (const void**)&m));
  OutView ov[1];
  CK(out_dev(counts, (size_t)ctx->T * (M + 1) * sizeof(int64_t), ctx->st_counts, ov[0]));
  CK(launch_label_counts(a, side, m, M, (long long*)ov[0].dev, ctx->stream));
  ctx->kernels += 2;
  CK(finish_outputs(ctx, ov, 1));
  return MOREA_OK;
}

int morea_elasticity(morea_ctx* ctx, const uint8_t* masks, int M, const float* factors, float* c_delta) {
  if (!ctx) return MOREA_EINVAL;
  if (M < 0 || M > 8 || (M > 0 && !factors) || !c_delta) return fail(ctx, MOREA_EINVAL, "bad M / buffers");
  std::vector<int64_t> cnt((size_t)ctx->T * (M + 1));
  int rc = morea_label_counts(ctx, nullptr, 0, masks, M, cnt.data());
  if (rc) return rc;
  std::vector<float> f;
  CK(to_host(ctx, factors, (size_t)M, f));
  std::vector<float> c(ctx->T);
  for (int t = 0; t < ctx->T; t++) {  // E2, in the oracle's order
    int64_t tot = 0;
    double acc = 0.0;
    for (int b = 0; b <= M; b++) {
      const int64_t n = cnt[(size_t)t * (M + 1) + b];
      tot += n;
      acc += (double)n * (b == 0 ? 1.0 : (double)f[b - 1]);
    }
    c[t] = tot > 0 ? (float)(acc / (double)tot) : 1.0f;
  }
  if (is_device_ptr(c_delta)) {
    CK(cudaMemcpyAsync(c_delta, c.data(), c.size() * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
  } else {
    std::memcpy(c_delta, c.data(), c.size() * sizeof(float));
  }
  return MOREA_OK;
}

int morea_dvf(morea_ctx* ctx, const float* offsets_one, int side, float* dvf, uint8_t* coverage) {
  NvtxScope nvtx_("morea_dvf");
  int rc = check_ready(ctx);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  if ((side != 0 && side != 1) || !dvf) return fail(ctx, MOREA_EINVAL, "bad side / buffers");
  EvalArgs a;
  rc = export_args(ctx, offsets_one, a);
  if (rc) return rc;
  OutView ov[2];
  CK(out_dev(dvf, (size_t)ctx->V * 3 * sizeof(float), ctx->st_dvf, ov[0]));
  CK(ctx->st_cov.ensure((size_t)ctx->V));
  CK(out_dev(coverage, (size_t)ctx->V, ctx->st_cov, ov[1]));
  unsigned char* cov = ov[1].dev ? (unsigned char*)ov[1].dev : ctx->st_cov.as<unsigned char>();
  CK(ctx->scratch_owner.ensure((size_t)ctx->V * sizeof(int)));
  CK(launch_dvf(a, side, ctx->scratch_owner.as<int>(), (float*)ov[0].dev, cov, ctx->stream));
  ctx->kernels += 4;
  CK(finish_outputs(ctx, ov, 2));
  return MOREA_OK;
}

// in/out array: device view, host arrays staged in and (by finish_outputs) back out
static cudaError_t inout_dev(morea_ctx* ctx, void* p, size_t bytes, DevBuf& st, OutView& v) {
  cudaError_t e = out_dev(p, bytes, st, v);
  if (e != cudaSuccess || !v.copy) return e;
  return cudaMemcpyAsync(v.dev, p, bytes, cudaMemcpyHostToDevice, ctx->stream);
}

int morea_mix_class(morea_ctx* ctx, int pop, float* offsets, morea_acc* acc, double* obj, double* tet_cache,
                    int n_groups, const int32_t* grp_off, const int32_t* changed_pts, const int32_t* cluster,
                    int n_clusters, const double* mu, const double* L, const uint8_t* fixed, int n_archive,
                    const double* archive, double steer_max, uint64_t seed, int64_t gen, int64_t sol_base,
                    uint8_t* accepted) {
  NvtxScope nvtx_("morea_mix_class");
  int rc = check_ready(ctx);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  if (pop < 0 || n_groups < 0 || !grp_off || n_clusters < 1 || n_archive < 0 || sol_base < 0)
    return fail(ctx, MOREA_EINVAL, "bad pop / groups / clusters / archive");
  if (pop > 0 && (!offsets || !acc || !obj || !tet_cache || !cluster || !mu || !L))
    return fail(ctx, MOREA_EINVAL, "null state or model");
  if (n_archive > 0 && !archive) return fail(ctx, MOREA_EINVAL, "null archive");
  Plan* Pp = nullptr;
  rc = get_plan(ctx, n_groups, grp_off, changed_pts, &Pp);
  if (rc) return rc;
  ctx->plan = Pp;
  const Plan& P = *Pp;
  if (!P.disjoint)
    return fail(ctx, MOREA_EINVAL, "the groups of morea_mix_class must be one colour class (pairwise disjoint "
                                   "changed points and dependent tets)");
  if (pop == 0 || n_groups == 0) return MOREA_OK;
  const int N = ctx->N, T = ctx->T, G = n_groups;
  // model layout: per cluster, mu_g (d_g) then the next group's; L_g (d_g^2) likewise
  std::vector<long long> moff(2 * G);
  long long mu_stride = 0, L_stride = 0;
  for (int g = 0; g < G; g++) {
    const long long d = 6LL * (P.key_off[g + 1] - P.key_off[g]);
    if (d > kMixMaxDimHost) return fail(ctx, MOREA_EINVAL, "FOS element %d has more than 32 points", g);
    moff[2 * g] = mu_stride;
    moff[2 * g + 1] = L_stride;
    mu_stride += d;
    L_stride += d * d;
  }
  std::vector<int32_t> cl;
  CK(to_host(ctx, cluster, (size_t)pop, cl));
  for (int k = 0; k < pop; k++)
    if (cl[k] < 0 || cl[k] >= n_clusters) return fail(ctx, MOREA_EINVAL, "cluster[%d] out of range", k);
  OutView ov[5];
  CK(inout_dev(ctx, offsets, (size_t)pop * N * 6 * sizeof(float), ctx->mx_off, ov[0]));
  CK(inout_dev(ctx, acc, (size_t)pop * sizeof(morea_acc), ctx->mx_acc, ov[1]));
  CK(inout_dev(ctx, obj, (size_t)pop * 3 * sizeof(double), ctx->mx_obj, ov[2]));
  CK(inout_dev(ctx, tet_cache, (size_t)pop * T * 4 * sizeof(double), ctx->mx_cache, ov[3]));
  CK(ctx->mx_accepted.ensure((size_t)pop * G));
  CK(out_dev(accepted, (size_t)pop * G, ctx->mx_accepted, ov[4]));
  unsigned char* acc_flags = ov[4].dev ? (unsigned char*)ov[4].dev : ctx->mx_accepted.as<unsigned char>();
  const int* cl_d = nullptr;
  const double *mu_d = nullptr, *L_d = nullptr, *ar_d = nullptr;
  const unsigned char* fx_d = nullptr;
  CK(in_dev(ctx, cluster, (size_t)pop * sizeof(int32_t), ctx->mx_cluster, (const void**)&cl_d));
  CK(in_dev(ctx, mu, (size_t)n_clusters * mu_stride * sizeof(double), ctx->mx_mu, (const void**)&mu_d));
  CK(in_dev(ctx, L, (size_t)n_clusters * L_stride * sizeof(double), ctx->mx_L, (const void**)&L_d));
  CK(in_dev(ctx, archive, (size_t)n_archive * 3 * sizeof(double), ctx->mx_arch, (const void**)&ar_d));
  CK(in_dev(ctx, fixed, (size_t)N * 3, ctx->mx_fixed, (const void**)&fx_d));
  CK(ctx->mx_moff.ensure(moff.size() * sizeof(long long)));
  CK(cudaMemcpyAsync(ctx->mx_moff.p, moff.data(), moff.size() * sizeof(long long), cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(ctx->mx_nv.ensure(std::max<size_t>(1, (size_t)pop * P.S * 6) * sizeof(float)));
  CK(ctx->mx_pobj.ensure((size_t)pop * G * 3 * sizeof(double)));
  CK(ctx->mx_pacc.ensure((size_t)pop * G * sizeof(morea_acc)));
  CK(ctx->mx_dep.ensure(std::max<size_t>(1, (size_t)pop * P.n_entries * 4) * sizeof(double)));
  CK(ctx->mx_base.ensure((size_t)pop * sizeof(morea_acc)));
  // M1-M3: sample every (solution, group) of the class
  MixArgs m;
  m.P = pop; m.G = G; m.N = N; m.T = T; m.S_total = P.S; m.n_entries = P.n_entries;
  m.sol_base = sol_base;
  m.offsets = (const float*)ov[0].dev;
  m.new_vals = ctx->mx_nv.as<float>();
  m.grp_off = P.grp_off;
  m.changed = P.changed;
  m.model_off = ctx->mx_moff.as<long long>();
  m.mu_stride = mu_stride;
  m.L_stride = L_stride;
  m.cluster = cl_d;
  m.mu = mu_d;
  m.L = L_d;
  m.fixed = fx_d;
  m.seed = seed;
  m.gen = gen;
  CK(launch_mix_sample(m, ctx->stream));
  ctx->kernels++;
  // a8: every candidate against the class-start state, with the per-tet cache
  CK(cudaMemcpyAsync(ctx->mx_base.p, ov[1].dev, (size_t)pop * sizeof(morea_acc), cudaMemcpyDeviceToDevice,
                     ctx->stream));
  CK(partial_core(ctx, P, pop, G, (const float*)ov[0].dev, ctx->mx_base.as<morea_acc>(), ctx->mx_nv.as<float>(),
                  (const double*)ov[3].dev, ctx->mx_pobj.as<double>(), ctx->mx_pacc.as<morea_acc>(),
                  ctx->mx_dep.as<double>()));
  // M4-M6: acceptance in group order, then commit
  CK(launch_mix_accept(pop, G, T, ctx->mx_base.as<morea_acc>(), ctx->mx_pacc.as<morea_acc>(),
                       (morea_acc*)ov[1].dev, (double*)ov[2].dev, ar_d, n_archive, steer_max, acc_flags,
                       ctx->stream));
  CK(launch_mix_commit(pop, G, N, T, P.S, P.n_entries, acc_flags, P.grp_off, P.changed,
                       P.group_off, P.canon_tet, ctx->mx_nv.as<float>(),
                       ctx->mx_dep.as<double>(), (float*)ov[0].dev, (double*)ov[3].dev, ctx->stream));
  ctx->kernels += 2;
  CK(finish_outputs(ctx, ov, 5));
  return MOREA_OK;
}

int morea_partial_deps(morea_ctx* ctx, int cap, int32_t* tets, int off_cap, int32_t* dep_off) {
  if (!ctx) return MOREA_EINVAL;
  if (!ctx->plan) return fail(ctx, MOREA_ESTATE, "no partial plan yet");
  const Plan& P = *ctx->plan;
  if (tets)
    for (int i = 0; i < std::min<int>(cap, (int)P.dep_tets.size()); i++) tets[i] = P.dep_tets[i];
  if (dep_off)
    for (int g = 0; g <= std::min(P.G, off_cap - 1); g++) dep_off[g] = P.dep_off[g];
  return (int)P.dep_tets.size();
}

int morea_partial_groups(const morea_ctx* ctx) {
  if (!ctx) return MOREA_EINVAL;
  return ctx->plan ? ctx->plan->G : MOREA_ESTATE;
}

int morea_check_folds(morea_ctx* ctx, int pop, const float* offsets, int32_t* fold_count,
                      double* severity, uint8_t* tet_flags) {
  NvtxScope nvtx_("morea_check_folds");
  int rc = check_ready(ctx);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  if (pop < 0 || (pop > 0 && !offsets)) return fail(ctx, MOREA_EINVAL, "bad pop / offsets");
  if (pop == 0) return MOREA_OK;
  const float* off = nullptr;
  CK(in_dev(ctx, offsets, (size_t)pop * ctx->N * 6 * sizeof(float), ctx->st_off, (const void**)&off));
  OutView ov[3];
  CK(out_dev(fold_count, (size_t)pop * sizeof(int32_t), ctx->st_i32, ov[0]));
  CK(out_dev(severity, (size_t)pop * sizeof(double), ctx->st_f64, ov[1]));
  CK(out_dev(tet_flags, (size_t)pop * 2 * ctx->T, ctx->st_u8, ov[2]));
  CK(launch_check_folds(mesh_of(ctx), ctx->sp, pop, off, (int*)ov[0].dev, (double*)ov[1].dev,
                        (unsigned char*)ov[2].dev, ctx->stream));
  ctx->kernels++;
  CK(finish_outputs(ctx, ov, 3));
  return MOREA_OK;
}

int morea_owner_map(morea_ctx* ctx, const float* offsets_one, int side, int32_t* owner) {
  NvtxScope nvtx_("morea_owner_map");
  int rc = check_ready(ctx);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  if (!offsets_one || !owner || (side != 0 && side != 1)) return fail(ctx, MOREA_EINVAL, "bad args");
  const float* off = nullptr;
  CK(in_dev(ctx, offsets_one, (size_t)ctx->N * 6 * sizeof(float), ctx->st_off, (const void**)&off));
  OutView ov[1];
  CK(out_dev(owner, (size_t)ctx->V * sizeof(int32_t), ctx->st_i32, ov[0]));
  EvalArgs a;
  std::memset(&a, 0, sizeof(a));
  a.vol = volumes_of(ctx);
  a.mesh = mesh_of(ctx);
  a.P = 1;
  a.offsets = off;
  plan_args(ctx, *ctx->full, a);
  a.sampler = MOREA_SAMPLER_VOXEL;
  a.n_setup_versions = 1;
  a.n_raster_versions = 1;
  a.expect[0] = a.expect[1] = -1;
  CK(eval_scratch(ctx, a));
  CK(launch_owner_map(a, side, (int*)ov[0].dev, ctx->stream));
  ctx->kernels += 3;
  CK(finish_outputs(ctx, ov, 1));
  return MOREA_OK;
}

int morea_sample_map(morea_ctx* ctx, const float* offsets_one, int side, float* h, uint8_t* fg) {
  NvtxScope nvtx_("morea_sample_map");
  int rc = check_ready(ctx);
  if (rc) return rc;
  CK(cudaSetDevice(ctx->device));
  if (!offsets_one || !h || !fg || (side != 0 && side != 1)) return fail(ctx, MOREA_EINVAL, "bad args");
  if (ctx->sampler != MOREA_SAMPLER_VOXEL) return fail(ctx, MOREA_ESTATE, "morea_sample_map needs the voxel sampler");
  const float* off = nullptr;
  ctx->host_in = false;
  CK(in_dev(ctx, offsets_one, (size_t)ctx->N * 6 * sizeof(float), ctx->st_off, (const void**)&off));
  OutView ov[2];
  CK(out_dev(h, (size_t)ctx->V * sizeof(float), ctx->st_f64, ov[0]));
  CK(out_dev(fg, (size_t)ctx->V, ctx->st_u8, ov[1]));
  CK(launch_fill((float*)ov[0].dev, (unsigned char*)ov[1].dev, ctx->V, ctx->stream));
  EvalArgs a;
  std::memset(&a, 0, sizeof(a));
  a.vol = volumes_of(ctx);
  a.mesh = mesh_of(ctx);
  a.P = 1;
  a.offsets = off;
  plan_args(ctx, *ctx->full, a);
  a.n_setup_versions = 1;
  a.n_raster_versions = 1;
  a.expect[0] = a.expect[1] = -1;
  a.dump_h = (float*)ov[0].dev;
  a.dump_fg = (unsigned char*)ov[1].dev;
  a.dump_side = side;
  CK(run_eval(ctx, a));
  ctx->kernels++;
  CK(finish_outputs(ctx, ov, 2));
  return MOREA_OK;
}

int morea_distance_map(morea_ctx* ctx, int side, int pair, float* out) {
  if (!ctx) return MOREA_EINVAL;
  CK(cudaSetDevice(ctx->device));
  if (!ctx->have_images) return fail(ctx, MOREA_ESTATE, "no images");
  if (side < 0 || side > 1 || pair < 0 || pair >= ctx->K || !out) return fail(ctx, MOREA_EINVAL, "bad args");
  CK(cudaMemcpyAsync(out, ctx->dmap[side].as<float>() + (size_t)pair * ctx->V, ctx->V * sizeof(float),
                     cudaMemcpyDefault, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return MOREA_OK;
}

int64_t morea_kernel_launches(const morea_ctx* ctx) { return ctx ? ctx->kernels : -1; }

int morea_prof_enable(morea_ctx* ctx, int on) {
  if (!ctx) return MOREA_EINVAL;
  ctx->prof = on != 0;
  return MOREA_OK;
}

int morea_prof_read(morea_ctx* ctx, int64_t* launches, double* ms, int64_t* samples,
                    int64_t* band_entries, int64_t* items, int64_t* skipped) {
  if (!ctx) return MOREA_EINVAL;
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  double tot = 0.0;
  for (auto& p : ctx->evs) {
    float m = 0.f;
    cudaEventElapsedTime(&m, p.first, p.second);
    tot += m;
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  ctx->evs.clear();
  unsigned long long st[4] = {0, 0, 0, 0};
  CK(cudaMemcpy(st, ctx->stats.p, sizeof(st), cudaMemcpyDeviceToHost));
  CK(cudaMemset(ctx->stats.p, 0, sizeof(st)));
  if (launches) *launches = ctx->prof_launches;
  if (ms) *ms = tot;
  if (samples) *samples = (int64_t)st[0];
  if (band_entries) *band_entries = (int64_t)st[1];
  if (items) *items = (int64_t)st[2];
  if (skipped) *skipped = (int64_t)st[3];
  ctx->prof_launches = 0;
  return MOREA_OK;
}

}  // extern "C"

// morea_sobol.cuh -- NEXT-1: the Sobol-in-tetrahedron sampler of PAPER.md
// App. A.2 (L744-751) on sm_100a, included by morea_kernels.cu (one TU).
//
// "We uniformly sample N points in each tetrahedron using its barycentric
// coordinate system, with N being determined by the volume of the tetrahedron.
// For each point, we sample 4 random real numbers r_i in [0;1] and take
// -log(r_i) ... normalize the coordinates by their sum ... the Sobol sequence
// ... seeding the Sobol sequence for each tetrahedron with a seed derived from
// its coordinates."  Readings S1..S9: DESIGN.md §3.
//
// k_setup writes a SobolRec per (item, side) (build_sobol).  k_sobol: persistent
// warps over the same item queue as k_raster; lane l of a 32-sample step takes
// point k = s0 + l.  In Gray-code order point k is x(g(k)) with g(k) = k ^ k>>1
// and x linear over GF(2) in g, so x(g(s0 + l)) = x(g(s0)) ^ x(g(l)) for s0 a
// multiple of 32: one warp XOR-reduction per step (x(g(s0))) and a per-lane
// constant (x(g(l))).
//
// Fast path in fp32: u = (x + 1/2) 2^-32, e = -lg2 u (MUFU.LG2), lambda = e / sum e
// (the ln 2 factor cancels), positions by fma chains.  Every decision the
// oracle takes on a position (clamp, floor, "is an integer") is taken from the
// fp32 position only when it is farther than a derived bound eps from every
// lattice plane; otherwise exact_sobol recomputes the position with the
// oracle's exact sequence of IEEE fp64 operations (the same -log routine, S5)
// and decides there.  Values (a, b, the guidance terms) stay fp32.
#pragma once

namespace morea {

// ---------------------------------------------------------------------------
// S8 exact fallback: lambda and both positions with the oracle's fp64 operation
// sequence; fa / fb = "some contributing corner (O5 clamp rules) is > 0".
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool sb_positive_at(const float* __restrict__ vol, const double x[3],
                                               int nx, int ny, int nz) {
  const int dims[3] = {nx, ny, nz};
  int lo[3], hi[3];  // contributing corner indices per axis (lo == hi: one corner)
#pragma unroll
  for (int a = 0; a < 3; a++) {
    const int n = dims[a];
    if (x[a] <= 0.0) {
      lo[a] = hi[a] = 0;
    } else if (x[a] >= (double)(n - 1)) {
      lo[a] = hi[a] = n - 1;
    } else {
      const double fl = floor(x[a]);
      lo[a] = (int)fl;
      hi[a] = (x[a] == fl) ? lo[a] : lo[a] + 1;
    }
  }
  // the (up to) 8 contributing corners, loaded together (one latency), then OR-ed
  bool any = false;
#pragma unroll
  for (int c = 0; c < 8; c++) {
    const int i = (c & 1) ? hi[0] : lo[0], j = (c & 2) ? hi[1] : lo[1], k = (c & 4) ? hi[2] : lo[2];
    any = any | (__ldg(&vol[((long long)k * ny + j) * nx + i]) > 0.0f);
  }
  return any;
}

__device__ __noinline__ void exact_sobol(const SobolRec& R, const unsigned xm[4], const float* volS,
                                         const float* volO, int nx, int ny, int nz, bool& fa,
                                         bool& fb) {
  double e[4];
  for (int j = 0; j < 4; j++) e[j] = sb_neg_log(xm[j]);
  const double s = __dadd_rn(__dadd_rn(__dadd_rn(e[0], e[1]), e[2]), e[3]);
  double lam[4];
  for (int j = 0; j < 4; j++) lam[j] = __ddiv_rn(e[j], s);
  double p[3], tp[3];
  for (int a = 0; a < 3; a++) {
    const double x0 = (double)R.Q[0][a] / 1024.0, y0 = (double)R.Qo[0][a] / 1024.0;
    const double d1 = (double)(R.Q[1][a] - R.Q[0][a]) / 1024.0;
    const double d2 = (double)(R.Q[2][a] - R.Q[0][a]) / 1024.0;
    const double d3 = (double)(R.Q[3][a] - R.Q[0][a]) / 1024.0;
    const double o1 = (double)(R.Qo[1][a] - R.Qo[0][a]) / 1024.0;
    const double o2 = (double)(R.Qo[2][a] - R.Qo[0][a]) / 1024.0;
    const double o3 = (double)(R.Qo[3][a] - R.Qo[0][a]) / 1024.0;
    p[a] = __dadd_rn(x0, __dadd_rn(__dadd_rn(__dmul_rn(lam[1], d1), __dmul_rn(lam[2], d2)),
                                   __dmul_rn(lam[3], d3)));
    tp[a] = __dadd_rn(y0, __dadd_rn(__dadd_rn(__dmul_rn(lam[1], o1), __dmul_rn(lam[2], o2)),
                                    __dmul_rn(lam[3], o3)));
  }
  fa = sb_positive_at(volS, p, nx, ny, nz);
  fb = sb_positive_at(volO, tp, nx, ny, nz);
}

// ---------------------------------------------------------------------------
// k_sobol
// ---------------------------------------------------------------------------
constexpr int kSbQueueCap = 64;  // < 32 pending + one step of <= 32
struct SobolWarp {
  SobolRec R;
  unsigned long long stat[4];
  uint4 qx[kSbQueueCap];  // Sobol states (x0..x3) of the points that are not proven quiet
};

// Item-side radius of the per-point empty-space test (see sobol_quiet): Rq = ceil(m) + 3,
// m = max |Qo - Q| / 1024 over the vertices and axes
__device__ __forceinline__ int sobol_radius(const SobolRec& R) {
  int mU = 0;
#pragma unroll
  for (int k = 0; k < 4; k++)
#pragma unroll
    for (int a = 0; a < 3; a++) mU = max(mU, abs(R.Qo[k][a] - R.Q[k][a]));
  return (mU + 1023) / 1024 + 3;
}

// Empty space, one side of an item: true when every voxel a point
// of the tet or its image can read is quiet -- background (I = 0) with no band entry
// on this side, and the other volume zero within Chebyshev radius Rq - 1.  The points
// lie in the bbox of the side's vertices and read the corners of their cells, so the
// box [floor(min) - 1, floor(max) + 2] covers every own footprint (and the cells the
// guidance prefilter reads).  An image is T(p) = p + sum_k l_k U_k with |U_k| <= m
// (Chebyshev), so its cell corners lie within 1 + m + 1 of any own corner of p's cell,
// plus rounding: Rq = ceil(m) + 3.  Then a = b = 0 and every distance is >= r at every
// point, so h = g = 0 for all N points, exactly.  Every image row (y, z) of the box
// must have its x range outside the row's hull of non-quiet voxels at Rq (one 4-byte
// load per row), early exit on the first miss.
__device__ __forceinline__ bool sobol_quiet(const SobolRec& R, const Volumes& V, int side, int lane) {
  const short2* qh = side == 0 ? V.qhull[0] : V.qhull[1];
  if (!qh) return false;
  const int dims[3] = {V.nx, V.ny, V.nz};
  int lo[3], hi[3];
#pragma unroll
  for (int a = 0; a < 3; a++) {
    int qmin = R.Q[0][a], qmax = R.Q[0][a];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      qmin = min(qmin, R.Q[k][a]);
      qmax = max(qmax, R.Q[k][a]);
    }
    lo[a] = max((qmin >> 10) - 1, 0);
    hi[a] = min((qmax >> 10) + 2, dims[a] - 1);
    if (lo[a] > hi[a]) return false;
  }
  const int Rq = sobol_radius(R);
  if (Rq > kQuietRmax) return false;  // beyond the radii the hulls carry
  const short2* h = qh + (Rq - kQuietRmin) * V.ny * V.nz;
  const int nyb = hi[1] - lo[1] + 1;
  const int nrows = nyb * (hi[2] - lo[2] + 1);
  for (int r0 = 0; r0 < nrows; r0 += 32) {
    const int r = r0 + lane;
    bool miss = false;
    if (r < nrows) {
      const int z = lo[2] + r / nyb, y = lo[1] + r % nyb;
      const short2 hb = __ldg(&h[z * V.ny + y]);
      miss = !(hi[0] < hb.x || lo[0] > hb.y);
    }
    if (__any_sync(FULLMASK, miss)) return false;
  }
  return true;
}

__device__ __forceinline__ float sb_plerp(float a, float b, float t, float omt) {
  return fmaf(t, b, omt * a);  // positivity-exact lerp (see plerp)
}

// corner, weights and texel coordinates of one position (O5 clamp), and the
// ambiguity test |f - 1/2| >= 1/2 - eps on every axis
struct SbPos {
  float fx, fy, fz;  // weights of the upper corners
  float ix, iy, iz;  // lower corner (clamped, exact floats)
};

// (x, y, z): position minus the integer offset i0 (floor of the tet's first vertex)
__device__ __forceinline__ bool sb_locate(float x, float y, float z, const float* i0, float eps,
                                          bool clamp, const Volumes& V, SbPos& P) {
  const float flx = floorf(x), fly = floorf(y), flz = floorf(z);
  P.fx = x - flx;
  P.fy = y - fly;
  P.fz = z - flz;
  const float lim = 0.5f - eps;
  const bool amb = (fabsf(P.fx - 0.5f) >= lim) | (fabsf(P.fy - 0.5f) >= lim) | (fabsf(P.fz - 0.5f) >= lim);
  P.ix = flx + i0[0];
  P.iy = fly + i0[1];
  P.iz = flz + i0[2];
  if (clamp) {
    P.fx = P.ix < 0.f ? 0.f : (P.ix > V.fnx2 ? 1.f : P.fx);
    P.fy = P.iy < 0.f ? 0.f : (P.iy > V.fny2 ? 1.f : P.fy);
    P.fz = P.iz < 0.f ? 0.f : (P.iz > V.fnz2 ? 1.f : P.fz);
    P.ix = fminf(fmaxf(P.ix, 0.f), V.fnx2);
    P.iy = fminf(fmaxf(P.iy, 0.f), V.fny2);
    P.iz = fminf(fmaxf(P.iz, 0.f), V.fnz2);
  }
  return amb;
}

// h from the values and the exact cases (S8)
__device__ __forceinline__ float sb_h(float a, float b, bool fa, bool fb) {
  return (fa && fb) ? (a - b) * (a - b) : ((!fa && !fb) ? 0.f : 1.f);
}

// all lanes call it (warp-uniform branch) and get h; lanes with ex = true take
// the cases from the exact fp64 positions.  a and b are arguments, so no value
// stays live across the call.
__device__ __noinline__ float exact_sobol_h(bool ex, float a, float b, const SobolRec& R, unsigned x0, unsigned x1,
                                            unsigned x2, unsigned x3, const Volumes& V, int side) {
  bool fa = a > 0.f, fb = b > 0.f;
  if (ex) {
    const unsigned xm[4] = {x0, x1, x2, x3};
    exact_sobol(R, xm, V.I[side], V.I[1 - side], V.nx, V.ny, V.nz, fa, fb);
  }
  return sb_h(a, b, fa, fb);
}

// -log2 u, u = (x + 1/2) 2^-32 >= 2^-33 (a normal float): MUFU.LG2 without the
// compiler's denormal fix-up (ftz changes nothing for normal inputs)
__device__ __forceinline__ float sb_neg_lg2(unsigned x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaf((float)x, 0x1.0p-32f, 0x1.0p-33f)));
  return -r;
}

// O5 clamp of a located position (corner into [0, n-2], weights 0 / 1 outside)
__device__ __forceinline__ void sb_clamp(const Volumes& V, SbPos& P) {
  P.fx = P.ix < 0.f ? 0.f : (P.ix > V.fnx2 ? 1.f : P.fx);
  P.fy = P.iy < 0.f ? 0.f : (P.iy > V.fny2 ? 1.f : P.fy);
  P.fz = P.iz < 0.f ? 0.f : (P.iz > V.fnz2 ? 1.f : P.fz);
  P.ix = fminf(fmaxf(P.ix, 0.f), V.fnx2);
  P.iy = fminf(fmaxf(P.iy, 0.f), V.fny2);
  P.iz = fminf(fmaxf(P.iz, 0.f), V.fnz2);
}

// SobolRec bit 2 keeps every vertex 2 kSbPadEps inside (-1, n); a sample whose
// fp32 error bound exceeds kSbPadEps is clamped
constexpr float kSbPadEps = 0x1.0p-5f;

template <bool TEX>
__device__ __forceinline__ float sb_trilinear(const Volumes& V, unsigned long long tex,
                                              const float* __restrict__ vol, float uoff,
                                              const SbPos& P) {
  const float gx = 1.f - P.fx, gy = 1.f - P.fy, gz = 1.f - P.fz;
  if (TEX) {
    // gather order (x0y1, x1y1, x1y0, x0y0); z first in packed fp32x2 on the aligned
    // pairs .xy / .zw, then y, then x (positivity-exact lerps, like k_raster)
    const float u = P.ix + uoff, v = fmaf(P.iz, V.fnyp, P.iy) + V.voff;
    const float4 g0 = tex2Dgather<float4>((cudaTextureObject_t)tex, u, v, 0);
    const float4 g1 = tex2Dgather<float4>((cudaTextureObject_t)tex, u, v + V.fnyp, 0);
    const float2 tz = make_float2(P.fz, P.fz), oz = make_float2(gz, gz);
    const float2 y1 = __ffma2_rn(tz, make_float2(g1.x, g1.y), __fmul2_rn(oz, make_float2(g0.x, g0.y)));
    const float2 y0 = __ffma2_rn(tz, make_float2(g1.z, g1.w), __fmul2_rn(oz, make_float2(g0.z, g0.w)));
    return sb_plerp(sb_plerp(y0.y, y1.x, P.fy, gy), sb_plerp(y0.x, y1.y, P.fy, gy), P.fx, gx);
  }
  float c[8];
  {
    // plain loads; the corner indices are clamped into the volume (only ambiguous
    // samples at the border can ask for index -1 or n, with weight ~0)
    const int x0 = min(max((int)P.ix, 0), V.nx - 2), y0 = min(max((int)P.iy, 0), V.ny - 2),
              z0 = min(max((int)P.iz, 0), V.nz - 2);
    const long long sy = V.nx, sz = (long long)V.nx * V.ny;
    const float* b = vol + z0 * sz + y0 * sy + x0;
    c[0] = __ldg(b); c[1] = __ldg(b + 1); c[2] = __ldg(b + sy); c[3] = __ldg(b + sy + 1);
    c[4] = __ldg(b + sz); c[5] = __ldg(b + sz + 1); c[6] = __ldg(b + sz + sy); c[7] = __ldg(b + sz + sy + 1);
  }
  return sb_plerp(sb_plerp(sb_plerp(c[0], c[1], P.fx, gx), sb_plerp(c[2], c[3], P.fx, gx), P.fy, gy),
                  sb_plerp(sb_plerp(c[4], c[5], P.fx, gx), sb_plerp(c[6], c[7], P.fx, gx), P.fy, gy),
                  P.fz, gz);
}

// one block of kSobolWarps warps per SM; the warps take consecutive items (the
// same tet for consecutive solutions) together, so their texel footprints share L1
constexpr int kSobolWarps = MOREA_SOBOL_WARPS;
constexpr int kSobolThreads = 32 * kSobolWarps;

template <bool TEX>
__global__ void __launch_bounds__(kSobolThreads, 1) k_sobol(const EvalArgs A) {
  __shared__ SobolWarp smem[kSobolWarps];
  __shared__ BlockQueue bq;
  bq.init();
  __shared__ unsigned sV[4][32];
  int warp, lane;
  asm volatile("shr.u32 %0, %1, 5;" : "=r"(warp) : "r"(threadIdx.x));
  asm volatile("and.b32 %0, %1, 31;" : "=r"(lane) : "r"(threadIdx.x));
  for (int t = threadIdx.x; t < 128; t += blockDim.x) sV[t >> 5][t & 31] = A.sobol_v[t];
  __syncthreads();
  SobolWarp& S = smem[warp];
  const Volumes& V = A.vol;
  // x(g(lane)): the per-lane constant part of the point index (S2)
  unsigned xlo[4];
  {
    const unsigned gl = (unsigned)lane ^ ((unsigned)lane >> 1);
#pragma unroll
    for (int j = 0; j < 4; j++) {
      unsigned v = 0;
#pragma unroll
      for (int b = 0; b < 5; b++)
        if ((gl >> b) & 1u) v ^= sV[j][b];
      xlo[j] = v;
    }
  }
  const long long per_v = (long long)A.n_entries * A.P;
  const long long n_items = per_v * A.n_raster_versions;
  if (lane == 0) S.stat[0] = S.stat[1] = S.stat[2] = S.stat[3] = 0ull;
  while (true) {
    const unsigned long long item = bq.claim(A.counter, lane, n_items, MOREA_CLAIM_CHUNK, MOREA_CLAIM_SPREAD);
    if ((long long)item >= n_items) break;
    const int ver = (int)(item / (unsigned long long)per_v);
    const long long rem = (long long)item - (long long)ver * per_v;
    const int es = (int)(rem / A.P);
    const int sol = (int)(rem - (long long)es * A.P);
    const int e = A.sched[es];
    const long long i = ((long long)ver * A.n_entries + e) * A.P + sol;
    // per-lane fp64 sums in local memory, touched once per flush (as in k_raster)
    double hg_local[2] = {0.0, 0.0};
    volatile double* hg = hg_local;
    long long n_tot = 0, n_side0 = 0;
    int nb = 0;
#pragma unroll 1
    for (int side = 0; side < 2; side++) {
      const int oth = 1 - side;
      constexpr int kVec = (int)(sizeof(SobolRec) / 16);
      __syncwarp();
      if (lane < kVec)
        reinterpret_cast<int4*>(&S.R)[lane] =
            __ldg(reinterpret_cast<const int4*>(&A.sgeom[2 * i + side]) + lane);
      __syncwarp();
      const SobolRec& R = S.R;
      if (!(R.flags & 1)) continue;
      const long long N = R.N;
      n_tot += N;
      if (side == 0) n_side0 = N;
      // empty space: h = g = 0 for every point (counted, not sampled); the fp64
      // test hook keeps every side on the sampling path
      if (!A.sobol_force_exact && sobol_quiet(R, V, side, lane)) {
        if (lane == 0) S.stat[3] += N;
        continue;
      }
      // O5 clamp only where a position can leave the range the gathers cover
      // exactly: [0, n-1] vertices for plain loads, (-1, n) (bit 2) on the
      // edge-padded textures; warp-uniform, so the common path skips the clamp
      const bool clamp = !(R.flags & ((TEX && kTexPad) ? 4 : 2));
      const unsigned m0 = R.mask[0] ^ xlo[0], m1 = R.mask[1] ^ xlo[1], m2 = R.mask[2] ^ xlo[2],
                     m3 = R.mask[3] ^ xlo[3];
      // (immediate offsets: cheap to rematerialise, so the compiler does not spill them)
      const float uoffS = TEX ? fmaf((float)side, V.fnxp, 1.0f + (float)kTexPad) : 1.0f;
      const float uoffO = TEX ? fmaf((float)oth, V.fnxp, 1.0f + (float)kTexPad) : 1.0f;
      // plain-load path only (TEX: the pointers are not kept live in the loop)
      const float* volS = TEX ? nullptr : (side == 0 ? V.I[0] : V.I[1]);
      const float* volO = TEX ? nullptr : (side == 0 ? V.I[1] : V.I[0]);
      const unsigned char* dil = side == 0 ? V.dil[0] : V.dil[1];
      float hf = 0.f, gf = 0.f;
      int step = 0;
      // One point per lane from its Sobol state (S2-S9): h and the guidance terms,
      // fp32 partial sums flushed into fp64 every 16 calls (warp-uniform)
      auto point = [&](unsigned x0, unsigned x1, unsigned x2, unsigned x3, bool valid) {
        // S5/S7 fast path: e = -lg2 u (the ln 2 factor cancels in the normalisation)
        const float e0 = sb_neg_lg2(x0), e1 = sb_neg_lg2(x1), e2 = sb_neg_lg2(x2), e3 = sb_neg_lg2(x3);
        const float sum = ((e0 + e1) + e2) + e3;
        const float rs = __frcp_rn(sum);
        const float l1 = e1 * rs, l2 = e2 * rs, l3 = e3 * rs;
        const float eps = fmaf(R.epsA, rs, R.epsB);
        const float px = fmaf(l3, R.D[2][0], fmaf(l2, R.D[1][0], fmaf(l1, R.D[0][0], R.x0[0])));
        const float py = fmaf(l3, R.D[2][1], fmaf(l2, R.D[1][1], fmaf(l1, R.D[0][1], R.x0[1])));
        const float pz = fmaf(l3, R.D[2][2], fmaf(l2, R.D[1][2], fmaf(l1, R.D[0][2], R.x0[2])));
        const float tx = fmaf(l3, R.Do[2][0], fmaf(l2, R.Do[1][0], fmaf(l1, R.Do[0][0], R.x0o[0])));
        const float ty = fmaf(l3, R.Do[2][1], fmaf(l2, R.Do[1][1], fmaf(l1, R.Do[0][1], R.x0o[1])));
        const float tz = fmaf(l3, R.Do[2][2], fmaf(l2, R.Do[1][2], fmaf(l1, R.Do[0][2], R.x0o[2])));
        SbPos Pp, Pt;
        bool amb;
        if (__all_sync(FULLMASK, !clamp)) {
          amb = sb_locate(px, py, pz, R.i0, eps, false, V, Pp);
          amb = sb_locate(tx, ty, tz, R.i0o, eps, false, V, Pt) || amb;
          // the no-clamp flag holds for positions within kSbPadEps of the exact
          // ones; a larger fp32 error bound (sum e tiny: never in practice) clamps
          if (__any_sync(FULLMASK, eps > kSbPadEps)) {
            if (eps > kSbPadEps) {
              sb_clamp(V, Pp);
              sb_clamp(V, Pt);
            }
          }
        } else {
          amb = sb_locate(px, py, pz, R.i0, eps, true, V, Pp);
          amb = sb_locate(tx, ty, tz, R.i0o, eps, true, V, Pt) || amb;
        }
        const float a = sb_trilinear<TEX>(V, V.texI, volS, uoffS, Pp);
        const float b = sb_trilinear<TEX>(V, V.texI, volO, uoffO, Pt);
        // h with both cases decided exactly (S8); the rare
        // exact path under a warp-uniform branch (no convergence barrier)
        const bool ex = (amb || A.sobol_force_exact) && valid;
        float h;
        if (__any_sync(FULLMASK, ex)) h = exact_sobol_h(ex, a, b, R, x0, x1, x2, x3, V, side);
        else h = sb_h(a, b, a > 0.f, b > 0.f);
        hf += valid ? h : 0.f;
        // a6 (S9): pairs whose distance can be < r in p's cell
        unsigned bm = 0u;
        if (V.K > 0 && valid) {
          const int cx = min(max((int)Pp.ix, 0), V.nx - 1), cy = min(max((int)Pp.iy, 0), V.ny - 1),
                    cz = min(max((int)Pp.iz, 0), V.nz - 1);
          bm = __ldg(&dil[((long long)cz * V.ny + cy) * V.nx + cx]);
        }
        nb += __popc(bm);
        while (__any_sync(FULLMASK, bm != 0u)) {
          if (bm) {
            const int pi = __ffs(bm) - 1;
            bm &= bm - 1;
            float d, Dp;
            if (TEX) {
              d = sb_trilinear<true>(V, V.texM, nullptr, fmaf((float)(side * V.K + pi), V.fnxp, 1.0f + (float)kTexPad), Pp);
              Dp = sb_trilinear<true>(V, V.texM, nullptr, fmaf((float)(oth * V.K + pi), V.fnxp, 1.0f + (float)kTexPad), Pt);
            } else {
              d = sb_trilinear<false>(V, 0ull, (side == 0 ? V.dmap[0] : V.dmap[1]) + (long long)pi * V.V,
                                      1.0f, Pp);
              Dp = sb_trilinear<false>(V, 0ull, (side == 0 ? V.dmap[1] : V.dmap[0]) + (long long)pi * V.V,
                                       1.0f, Pt);
            }
            if (d < V.rf) {
              const float dd = d - Dp;
              gf += __ldg(&V.wfd[side * kMaxPairs + pi]) * ((V.rf - d) + V.rlo) * (dd * dd);
            }
          }
        }
        if ((++step & 15) == 0) {
          hg[0] = hg[0] + (double)hf;
          hg[1] = hg[1] + (double)gf;
          hf = gf = 0.f;
        }
      };
      // Empty space per point: a point whose cell block (the
      // 4^3 voxels around floor(p), which hold its exact cell's corners while the
      // fp32 error is <= 1/2) is quiet at Rq has a = b = 0 and no distance < r,
      // so h = g = 0: it is counted (N) and not evaluated.  The others queue their
      // Sobol state and are evaluated 32 at a time.  The fp64 test hook keeps every
      // point on the evaluation path.
      const int Rq = sobol_radius(R);
      const unsigned char* qc =
          (!A.sobol_force_exact && Rq <= kQuietRmax) ? (side == 0 ? V.qcell[0] : V.qcell[1]) : nullptr;
      int qn = 0;  // queued points (warp-uniform)
      int nquiet = 0;
      // S2: x(g(s0)) ^ x(g(lane)) ^ mask, updated per step: for s0 = 32 m,
      // g(s0 + 32) ^ g(s0) = 2^4 ^ 2^(5 + ctz(m + 1)), so two direction numbers
      // per dimension change (warp-uniform)
      unsigned x0 = m0, x1 = m1, x2 = m2, x3 = m3;
      const int Ni = (int)N;  // < 2^31: k_setup flags larger counts (DOMAIN) and clears the side
#pragma unroll 1
      for (int s0 = 0;; s0 += 32) {
        const bool more = s0 < Ni;  // warp-uniform
        if (more) {
          if (s0 > 0) {
            const int b = 4 + __ffs(s0 >> 5);  // 5 + ctz(m + 1), m + 1 = s0 / 32
            x0 ^= sV[0][4] ^ sV[0][b];
            x1 ^= sV[1][4] ^ sV[1][b];
            x2 ^= sV[2][4] ^ sV[2][b];
            x3 ^= sV[3][4] ^ sV[3][b];
          }
          const bool valid = s0 + lane < Ni;
          bool live = valid;
          if (qc) {  // item-uniform
            const float e0 = sb_neg_lg2(x0), e1 = sb_neg_lg2(x1), e2 = sb_neg_lg2(x2), e3 = sb_neg_lg2(x3);
            const float rs = __frcp_rn(((e0 + e1) + e2) + e3);
            const float l1 = e1 * rs, l2 = e2 * rs, l3 = e3 * rs;
            const float eps = fmaf(R.epsA, rs, R.epsB);
            const float px = fmaf(l3, R.D[2][0], fmaf(l2, R.D[1][0], fmaf(l1, R.D[0][0], R.x0[0])));
            const float py = fmaf(l3, R.D[2][1], fmaf(l2, R.D[1][1], fmaf(l1, R.D[0][1], R.x0[1])));
            const float pz = fmaf(l3, R.D[2][2], fmaf(l2, R.D[1][2], fmaf(l1, R.D[0][2], R.x0[2])));
            const int cx = min(max((int)(floorf(px) + R.i0[0]), 0), V.nx - 1);
            const int cy = min(max((int)(floorf(py) + R.i0[1]), 0), V.ny - 1);
            const int cz = min(max((int)(floorf(pz) + R.i0[2]), 0), V.nz - 1);
            const bool quiet = eps <= 0.5f && (int)__ldg(&qc[(cz * V.ny + cy) * V.nx + cx]) >= Rq;
            nquiet += (valid && quiet) ? 1 : 0;
            live = valid && !quiet;
          }
          const unsigned lm = __ballot_sync(FULLMASK, live);
          if (live) S.qx[qn + __popc(lm & ((1u << lane) - 1u))] = make_uint4(x0, x1, x2, x3);
          qn += __popc(lm);
        }
        // evaluate 32 queued points, or at the end what is left (one call site)
        if (qn >= 32 || (!more && qn > 0)) {
          const int take = min(qn, 32);
          qn -= take;
          __syncwarp();
          const uint4 q = S.qx[qn + min(lane, take - 1)];
          __syncwarp();
          point(q.x, q.y, q.z, q.w, lane < take);
        }
        if (!more) break;
      }
      nquiet = warp_sum_i(nquiet);
      if (lane == 0) S.stat[3] += nquiet;
      hg[0] = hg[0] + (double)hf;
      hg[1] = hg[1] + (double)gf;
    }
    HGN out;
    out.h = warp_sum_d(hg[0]);
    out.g = warp_sum_d(hg[1]);
    out.n = n_tot;
    out.n0 = n_side0;
    const int nb_w = warp_sum_i(nb);
    if (lane == 0) {
      A.hgn[i] = out;
      S.stat[0] += n_tot;
      S.stat[1] += nb_w;
      S.stat[2] += 1;
      debug_count_item(A);
    }
  }
  debug_check_items(A, n_items);
  if (lane == 0 && A.stats) {
    atomicAdd(&A.stats[0], S.stat[0]);
    atomicAdd(&A.stats[1], S.stat[1]);
    atomicAdd(&A.stats[2], S.stat[2]);
    atomicAdd(&A.stats[3], S.stat[3]);
  }
}

int sobol_block_warps() { return kSobolWarps; }

int sobol_blocks_per_sm(bool tex) {
  int nb = 0;
  cudaError_t e = tex ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sobol<true>, kSobolThreads, 0)
                      : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sobol<false>, kSobolThreads, 0);
  if (e != cudaSuccess) return 1;
  return nb > 0 ? nb : 1;
}

cudaError_t launch_sobol(const EvalArgs& a, int grid, cudaStream_t s) {
  if (a.vol.use_tex) k_sobol<true><<<grid, kSobolThreads, 0, s>>>(a);
  else k_sobol<false><<<grid, kSobolThreads, 0, s>>>(a);
  return cudaGetLastError();
}

// dil[v] = OR of band[c] over the cell corners c in v + {0,1}^3 (clamped)
__global__ void k_dilate_band(const unsigned char* __restrict__ band, int nx, int ny, int nz,
                              unsigned char* __restrict__ dil) {
  const long long V = (long long)nx * ny * nz;
  for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < V;
       v += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(v % nx), y = (int)((v / nx) % ny), z = (int)(v / ((long long)nx * ny));
    unsigned m = 0;
    for (int dz = 0; dz < 2; dz++)
      for (int dy = 0; dy < 2; dy++)
        for (int dx = 0; dx < 2; dx++) {
          const int cx = min(x + dx, nx - 1), cy = min(y + dy, ny - 1), cz = min(z + dz, nz - 1);
          m |= band[((long long)cz * ny + cy) * nx + cx];
        }
    dil[v] = (unsigned char)m;
  }
}

cudaError_t launch_dilate_band(const unsigned char* band, int nx, int ny, int nz, unsigned char* dil,
                               cudaStream_t s) {
  const long long V = (long long)nx * ny * nz;
  const long long nblk = (V + 255) / 256;
  const int grid = (int)(nblk < 148 * 16 ? nblk : 148 * 16);
  k_dilate_band<<<grid, 256, 0, s>>>(band, nx, ny, nz, dil);
  return cudaGetLastError();
}

}  // namespace morea

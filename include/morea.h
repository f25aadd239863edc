/*
 * morea.h -- C-ABI of the B200-native MOREA hot path (arXiv 2303.04873).
 *
 * Batched evaluation of dual-dynamic tetrahedral-mesh deformations over a whole
 * MO-RV-GOMEA population: f_magnitude (§4.1.1, eq. L257-259),
 * f_intensity (§4.1.2, eq. L316-323), f_guidance (§4.1.3, eq. L338-342;
 * App. A.3) and signed-volume fold detection (§4.1.4; App. A.4
 * L806-810), as full evaluations and as GOMEA partial evaluations over the
 * tetrahedra that depend on a changed FOS point set (§1, §4.2.1
 * L399-410).  The readings of the paper that fix every ambiguous detail are
 * listed in DESIGN.md §3 (O1..O13); the short forms are repeated per call.
 *
 * Conventions common to every call
 *  - Positions are in voxel-index units: voxel (i,j,k) has its centre at
 *    (i,j,k).  Volumes are float32, x-fastest (index (k*ny + j)*nx + i).
 *  - Every buffer is caller-owned.  Unless a call says otherwise, an array
 *    argument may be HOST memory (pageable or pinned) or DEVICE memory of the
 *    context's device; the library detects which (cudaPointerGetAttributes).
 *    Host inputs are staged to device scratch inside the call and consumed
 *    before it returns (a call with a host input or a host output synchronises
 *    the context stream before returning), so the caller may reuse host
 *    buffers at once.  When every pointer is device memory the call is
 *    asynchronous and stream-ordered on the context stream (device offsets
 *    that are not 8-byte aligned are staged by a device copy).
 *  - A context is bound to one device and is not thread-safe.  Multi-GPU use
 *    is one context per process/rank; the library itself makes no NCCL calls.
 *  - Return value: MOREA_OK (0) or a negative MOREA_E* code; the message is
 *    available from morea_last_error().  Per-solution conditions are FLAGS in
 *    morea_acc.flags, never errors (a batch never fails for one solution).
 */
#ifndef MOREA_H
#define MOREA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ---- */
#define MOREA_OK 0
#define MOREA_EINVAL (-1)  /* bad shape/index/value, negative or NaN intensity */
#define MOREA_ESTATE (-2)  /* eval before morea_load_images / morea_set_mesh */
#define MOREA_EDOMAIN (-3) /* base point outside the Q.10 window or degenerate base tet */
#define MOREA_ECUDA (-4)   /* CUDA runtime error (message has the CUDA error string) */
#define MOREA_ENOMEM (-5)  /* device allocation failed */

/* ---- per-solution flags (morea_acc.flags) ---- */
#define MOREA_F_DOMAIN 1 /* some point outside the Q.10 window: objectives are NaN */
#define MOREA_F_EMPTY 2  /* no samples (n_samples == 0): objectives are NaN */
#define MOREA_F_COVERAGE 4 /* full evaluation only: on some side the number of owned voxel
                              centres differs from the base mesh's (row a9 coverage check:
                              a gap or an overlap, e.g. from moved hull points or a fold) */

/* ---- morea_set_mesh options ---- */
#define MOREA_SPOKE_FACE_CENTROID 0 /* spoke = vertex -> centroid of the opposite face (O9, default) */
#define MOREA_SPOKE_TET_CENTROID 1  /* spoke = tet centroid -> vertex (3/4 of the above) */

/* ---- morea_set_sampler modes ---- */
#define MOREA_SAMPLER_VOXEL 0 /* exactly-once voxel centres (north_star, O3; default) */
#define MOREA_SAMPLER_SOBOL 1 /* Sobol points per tet (App. A.2; NEXT-1) */

/* Q.10 window (reading O1): canonical coordinates Q = round-half-even(1024*B +
 * 1024*O) must satisfy -256*1024 <= Q < 768*1024 on every axis. */
#define MOREA_WINDOW_LO_VOX (-256)
#define MOREA_WINDOW_HI_VOX 768

typedef struct morea_ctx morea_ctx;

/* Per-solution accumulator (48 bytes).  Objectives derive from it as
 *   f_magnitude = m_sum / (10 T)      (L258)
 *   f_intensity = h_sum / n_samples   (L317, n_samples = |P_s| + |P_t|)
 *   f_guidance  = g_sum / n_samples   (L339)
 * folds = number of (tet, side) pairs whose exact signed volume has another
 * sign than the tet's reference sign (0 counts as a fold; App. A.4,
 * "either of the two meshes" §4.3.1); severity = sum of |signed volume|
 * in mm^3 over those pairs (L810).  folds > 0 means infeasible: objectives are
 * still written but voxels may be owned twice (or not at all). */
typedef struct {
    double h_sum, g_sum, m_sum, severity;
    int64_t n_samples;
    int32_t folds, flags;
} morea_acc;

/* Create a context on `cuda_device`.  `cuda_stream` (a cudaStream_t of that
 * device) is used for all work; NULL creates a context-owned stream that is
 * ordered with the legacy default stream (cudaStreamDefault flags), so inputs
 * written there before a call are visible to it.  With a caller stream the
 * caller orders its producers on that stream.  Returns MOREA_ECUDA if the
 * device is unusable. */
int morea_create(int cuda_device, void *cuda_stream, morea_ctx **out);
void morea_destroy(morea_ctx *ctx);
/* Message of the last failed call ("" if none).  Owned by the context. */
const char *morea_last_error(const morea_ctx *ctx);
/* The stream the context launches on (cudaStream_t as void*). */
void *morea_stream(const morea_ctx *ctx);

/* Load the two volumes and the contour guidance (one-off per problem).
 *  nx,ny,nz >= 2, <= 768; spacing_mm[3] > 0 (physical voxel size; lengths,
 *    distances, r and severities are in mm).
 *  I_s, I_t: V = nx*ny*nz float32 each, finite, >= 0, background exactly 0
 *    (h's zero/non-zero cases, L318-322; reading O6); non-zero values must be
 *    >= 2^-40 (~9.1e-13) so the fp32 interpolant of a non-zero footprint cannot
 *    underflow to 0 (the exact case split relies on it).
 *  n_pairs K in [0, 8]: pairs <C_s, C_t>_i of contour point sets (L332-333).
 *    cs_off/ct_off: K+1 int64 CSR offsets (non-decreasing, cs_off[0] = 0) into
 *    cs_xyz/ct_xyz: float32 xyz triples in voxel units.  Weights per side are
 *    |C_i| / |G_side| (L340).
 *  r_mm: truncation radius of the guidance term (App. A.3); <= 0 means
 *    0.025 * nx * spacing_mm[0] ("2.5% of the width of the image").
 * Builds on the device, in fp64 and exactly reproducibly: the distance maps
 * D_i^side(q) = min_c ||(q - c) * spacing|| (L793, brute force over all points,
 * rounded once to fp32) and the narrow-band masks bit i = [D_i^side(q) < r].
 * Synchronises the context stream. */
int morea_load_images(morea_ctx *ctx, int nx, int ny, int nz, const double spacing_mm[3],
                      const float *I_s, const float *I_t, int n_pairs, const int64_t *cs_off,
                      const float *cs_xyz, const int64_t *ct_off, const float *ct_xyz,
                      double r_mm);

/* Set the dual-dynamic mesh topology and its base positions (L397).
 *  base_xyz: N*3 float32 voxel units; tets: T*4 int32 point ids in [0, N);
 *  c_delta: T float32 elasticity factors (L253) or NULL for 1.0;
 *  spoke_mode: MOREA_SPOKE_FACE_CENTROID or MOREA_SPOKE_TET_CENTROID (O9).
 * Reference signs are the exact signs of the base tets (App. A.4); a base
 * point outside the Q.10 window or a zero-volume base tet is MOREA_EDOMAIN.
 * Requires morea_load_images first.  Synchronises the context stream. */
int morea_set_mesh(morea_ctx *ctx, int n_points, const float *base_xyz, int n_tets,
                   const int32_t *tets, const float *c_delta, int spoke_mode);

/* Full evaluation of `pop` solutions.
 *  offsets: pop*N*6 float32, per point (src dx,dy,dz, tgt dx,dy,dz): the point
 *    is at base + offset on each side (the genotype of L528, "transform-both"
 *    L2003).
 *  obj: pop*3 float64 (f_magnitude, f_intensity, f_guidance) or NULL;
 *  acc: pop morea_acc or NULL;
 *  tet_cache: NULL or pop*T*4 float64 receiving per-tet contributions
 *    {h, g, n_samples, m} summed over both sides -- the "old" values a later
 *    morea_eval_partial can reuse instead of recomputing them.
 * Samples are the voxel centres owned by each tet on each side under the exact
 * exactly-once rule (O3); a sample q of side s maps to x = T(q) by the tet's
 * barycentric coordinates (O4) and contributes h(I_s(q), trilinear(I_t, x))
 * (O5, O6) and, for each pair with D_i^s(q) < r, w_i (r - d)/r (d - D_i^t(x))^2
 * (O8); symmetrically for side t. */
int morea_eval_full(morea_ctx *ctx, int pop, const float *offsets, double *obj, morea_acc *acc,
                    double *tet_cache);

/* Partial (delta) evaluation of n_groups changed point sets per solution
 * (O10).  For group g, S_g = changed_pts[grp_off[g] .. grp_off[g+1]) (point
 * ids, no duplicates inside a group) and D_g = the tets incident to S_g.  The
 * result for (solution k, group g) is
 *     acc' = base_acc[k] - sum_{D_g} contrib(base) + sum_{D_g} contrib(new)
 * where "new" replaces the offsets of S_g by
 *     new_vals[(k*S + grp_off[g] + i)*6 + c],  S = grp_off[n_groups].
 * Groups are independent (each delta is taken against the base alone), so
 * groups may overlap; a colour class (disjoint D_g, L409-410) is the intended
 * use.  grp_off / changed_pts are HOST arrays (the static FOS structure; the
 * dependent-tet plan is built on the host and cached).  base_acc must be the
 * accumulator of base_offsets (caller's contract).
 *  tet_cache: NULL (old contributions are recomputed: 2x the work) or the
 *    pop*T*4 array written by morea_eval_full for base_offsets (bitwise equal
 *    results either way).
 *  obj: pop*n_groups*3, acc: pop*n_groups (index k*n_groups + g), either NULL.
 *  dep_cache_out: NULL or pop*ND*4 float64, ND = sum_g |D_g|: the new per-tet
 *    contributions {h, g, n, m} in group order, tets ascending within a group
 *    (see morea_partial_deps for the tet ids).
 * flags' = (base flags & DOMAIN) | DOMAIN if a new point leaves the window |
 * EMPTY if n_samples' == 0. */
int morea_eval_partial(morea_ctx *ctx, int pop, const float *base_offsets,
                       const morea_acc *base_acc, int n_groups, const int32_t *grp_off,
                       const int32_t *changed_pts, const float *new_vals, const double *tet_cache,
                       double *obj, morea_acc *acc, double *dep_cache_out);

/* Select the sample set of subsequent evaluations.
 *  MOREA_SAMPLER_VOXEL: the voxel centres each tet owns, exactly once (O3).
 *  MOREA_SAMPLER_SOBOL: PAPER.md App. A.2 "We uniformly sample N points
 *    in each tetrahedron using its barycentric coordinate system, with N being
 *    determined by the volume of the tetrahedron ... 4 random real numbers r_i
 *    ... -log(r_i) ... normalize the coordinates by their sum ... the Sobol
 *    sequence ... seeding the Sobol sequence for each tetrahedron with a seed
 *    derived from its coordinates."  Per (solution, tet, side):
 *    N = floor(rate |Delta| / (6 1024^3) + 1/2) (rate = samples per voxel of tet
 *    volume); point k = Gray-code Sobol point k (4 dims, Joe-Kuo directions)
 *    XOR-shifted by masks from FNV-1a of the side's Q.10 vertex coordinates;
 *    a = trilinear I_side(p) and b = trilinear I_other(T p), both interpolated;
 *    the guidance term uses d = trilinear D_i^side(p).  Readings S1..S9 in
 *    DESIGN.md §3.  f_int / f_guid normalise by the total sample count.  The
 *    coverage flag is not computed in this mode.
 * rate must be in (0, 8].  Per-side point counts are 32-bit: a (solution, tet)
 * whose count exceeds 2^31 - 1 (a tet of more than 2^31 / rate voxels, only
 * possible for degenerate meshes spanning most of the Q.10 window) gets
 * MOREA_F_DOMAIN and NaN objectives instead of a wrong count.  Takes effect for the following morea_eval_*
 * calls (morea_owner_map always uses the voxel-centre rasterizer).
 * Errors: EINVAL (bad mode / rate), ESTATE (before morea_create finished). */
int morea_set_sampler(morea_ctx *ctx, int mode, double rate);

/* Fold repair (§4.3.1): "For each
 * point in a folded tetrahedron, the method mutates the point using a Gaussian
 * distribution scaled by its estimated distance to the surrounding 3D polygon.
 * After 64 samples, the change with the best constraint improvement is
 * selected, if present.  If all samples result in a deterioration, repair is
 * aborted."  Per solution k, side s in {source, target}: the vertices of the
 * tets folded on s at the start of the pass, ascending; each gets 64 candidates
 * o' = o + sigma z (z ~ N(0, I3) from SplitMix64 keys of (seed, sol_base + k, s,
 * point, candidate), Marsaglia's polar method); sigma = 1/2 min distance (voxels)
 * to the opposite-face planes of its incident unfolded tets; a candidate scores
 * (folded incident tets, their severity) lexicographically; the best one is
 * applied iff it is strictly better, else the point is "aborted".  Readings
 * P1..P8 in DESIGN.md §3.  Deterministic for a given seed and sol_base.
 *  offsets: pop*N*6, updated in place (host or device).
 *  fixed: NULL or N*3 uint8, axes the repair must not move (both sides), e.g.
 *    hull points kept on their boundary planes.
 *  moved / aborted: NULL or pop int32: points moved / points without an
 *    improving candidate.
 * Re-run morea_check_folds for the remaining folds. */
int morea_repair(morea_ctx *ctx, int pop, float *offsets, const uint8_t *fixed, uint64_t seed,
                 int64_t sol_base, int32_t *moved, int32_t *aborted);

/* Optimal mixing of one FOS colour class on the device (
 * PAPER.md §3: "distributions are estimated for each FOS element in
 * each cluster, and new, partial solutions are sampled from these distributions.
 * Newly sampled partial solutions are evaluated and accepted if their insertion
 * into the parent solution results in a solution that dominates the parent
 * solution or that is non-dominated in the current elitist archive").
 * The groups (grp_off / changed_pts, HOST arrays as for morea_eval_partial) must
 * be one colour class: pairwise disjoint changed points and dependent tets
 * (checked: MOREA_EINVAL otherwise).  Per solution k and
 * group g: z ~ N(0, I_d) (d = 6 |S_g|, SplitMix64 keys of (seed, gen,
 * sol_base + k, g), Marsaglia's polar method); x = mu + L z with the model of
 * cluster[k] (mu: n_clusters blocks of sum_g d_g doubles, group after group; L:
 * n_clusters blocks of sum_g d_g^2 doubles, row-major lower triangles); the new
 * point values are fp32(x) (point order of changed_pts, then src xyz, tgt xyz),
 * axes flagged in `fixed` (NULL or N*3) keep the parent's value.  Each candidate
 * is evaluated partially (per-tet cache); groups are then accepted in id order,
 * each against the solution as updated by the earlier accepted groups: a
 * candidate with folds, a DOMAIN/EMPTY flag or (steer_max > 0) f_guidance >
 * steer_max is rejected; otherwise it is accepted iff it dominates the parent
 * or no archive member (n_archive x 3 objectives, fixed during the call)
 * dominates it.  Accepted groups are committed: offsets, acc, obj and the
 * tet_cache rows of their dependent tets.  Readings M1..M7 in DESIGN.md §3.
 *  offsets (pop*N*6), acc (pop), obj (pop*3), tet_cache (pop*T*4): the
 *    population state, updated in place (host or device; obj / acc / cache must
 *    be those of offsets, e.g. from morea_eval_full).
 *  accepted: NULL or pop*n_groups bytes.
 * Archive insertion and model estimation are the caller's. */
int morea_mix_class(morea_ctx *ctx, int pop, float *offsets, morea_acc *acc, double *obj, double *tet_cache,
                    int n_groups, const int32_t *grp_off, const int32_t *changed_pts, const int32_t *cluster,
                    int n_clusters, const double *mu, const double *L, const uint8_t *fixed, int n_archive,
                    const double *archive, double steer_max, uint64_t seed, int64_t gen, int64_t sol_base,
                    uint8_t *accepted);

/* Rasterizer reuse.
 * Object counts per tet (App. A.1: "We compute the overlap
 * that each object mask has with the tetrahedron ... which produces one fraction
 * per object"): for the solution offsets_one (N*6; NULL = the base mesh), the
 * voxel centres each tet owns on `side` (O3, exactly once) are counted per
 * label: masks is a V byte volume (x-fastest), bit m = object m (m < M <= 8);
 * a voxel's label is 1 + its lowest set bit (objects in priority order), 0 if
 * none.  counts: T*(M+1) int64 (host or device).  Readings E1..E3. */
int morea_label_counts(morea_ctx *ctx, const float *offsets_one, int side, const uint8_t *masks, int M,
                       int64_t *counts);
/* Elasticity factors (App. A.1: "These object fractions are multiplied
 * by pre-determined elasticity factors ... yielding an overall element-specific
 * factor"): c_delta[t] = sum_m frac_m factors[m] + (1 - sum_m frac_m) * 1.0 over
 * the base mesh's source-side voxel centres (1.0 for a tet owning none).  Feed
 * the result to morea_set_mesh.  c_delta: T floats, host or device. */
int morea_elasticity(morea_ctx *ctx, const uint8_t *masks, int M, const float *factors, float *c_delta);
/* Deformation vector field of one side (§5.4, "a forward and an inverse
 * DVF"): at every voxel centre q owned on `side` by some tet, T(q) - q in mm
 * (O4 with the exact numerator, bit-identical to the oracle; the lowest tet id
 * wins where a fold gives several owners); 0 elsewhere.  side 0 = forward
 * (source voxels), 1 = inverse.  dvf: V*3 float (x-fastest voxels, xyz per
 * voxel); coverage: NULL or V bytes, 1 where owned. */
int morea_dvf(morea_ctx *ctx, const float *offsets_one, int side, float *dvf, uint8_t *coverage);

/* The dependent tets of the plan of the last morea_eval_partial,
 * morea_mix_class or morea_prepare_partial call: writes up to `cap` tet ids
 * (group order, ascending within a group) into `tets` (host, or NULL) and up to
 * `off_cap` of the n_groups+1 offsets into `dep_off` (host, or NULL).
 * Returns ND (>= 0), or ESTATE if no plan exists yet. */
int morea_partial_deps(morea_ctx *ctx, int cap, int32_t *tets, int off_cap, int32_t *dep_off);
/* n_groups of that plan (>= 0), or ESTATE. */
int morea_partial_groups(const morea_ctx *ctx);

/* Build (or find) the dependent-tet plan of a partial request ahead of time
 * (same arguments as morea_eval_partial).  Plans are cached per distinct
 * (grp_off, changed_pts) request, least recently used first out of 64, so a
 * generation that evaluates every colour class in turn rebuilds nothing; a
 * miss builds the plan on the host and uploads it asynchronously (pinned
 * staging, no stream synchronisation).  Optional: morea_eval_partial builds
 * missing plans itself. */
int morea_prepare_partial(morea_ctx *ctx, int n_groups, const int32_t *grp_off, const int32_t *changed_pts);

/* Fold check only (row a9): per solution the number of folded (tet, side) pairs
 * and their summed severity (mm^3); tet_flags (NULL or pop*2*T uint8, index
 * (k*2 + side)*T + t) gets 1 for a folded pair.  fold_count/severity may be
 * NULL.  No voxel work. */
int morea_check_folds(morea_ctx *ctx, int pop, const float *offsets, int32_t *fold_count,
                      double *severity, uint8_t *tet_flags);

/* Test hook (not on the hot path): owning tet of every voxel of one side for
 * one solution, with the same rasterizer the evaluation uses.  owner: V int32,
 * tet id, -1 = no owner, -2 = more than one owner.  offsets_one: N*6. */
int morea_owner_map(morea_ctx *ctx, const float *offsets_one, int side, int32_t *owner);

/* Test hook (not on the hot path): the per-sample values of one side of one
 * solution from the evaluation kernel itself (k_sweep in a dump instantiation):
 * for every voxel centre q owned on `side`, h[q] = h(I_side(q), I_other(T(q)))
 * as summed into f_intensity (fp32) and fg[q] = the exact O6 case decision
 * (1: some contributing corner of the trilinear footprint is > 0); h = NaN,
 * fg = 255 where no tet owns q.  h: V float32, fg: V bytes.  Voxel sampler only. */
int morea_sample_map(morea_ctx *ctx, const float *offsets_one, int side, float *h, uint8_t *fg);

/* Test hook: the fp32 distance map D_pair^side (V floats) built by
 * morea_load_images. */
int morea_distance_map(morea_ctx *ctx, int side, int pair, float *out);

/* Profiling of the evaluation kernel (bench.py): when enabled, every launch of
 * the rasterize/evaluate kernel is bracketed by CUDA events on the context
 * stream and its algorithmic work is counted.  morea_prof_read synchronises
 * and returns: launches, summed kernel milliseconds, sampled voxels, band
 * entries, (tet, solution) items, and the samples counted without being
 * swept: voxel sampler, those of quiet rows (every voxel background with no
 * band entry and the other volume zero within the item's reach: h = g = 0
 * exactly); Sobol sampler, the points of quiet item sides.
 * Reading resets the counters. */
int morea_prof_enable(morea_ctx *ctx, int on);
/* Number of kernels this context has launched since it was created. */
int64_t morea_kernel_launches(const morea_ctx *ctx);
int morea_prof_read(morea_ctx *ctx, int64_t *launches, double *ms, int64_t *samples,
                    int64_t *band_entries, int64_t *items, int64_t *skipped);

#ifdef __cplusplus
}
#endif
#endif /* MOREA_H */

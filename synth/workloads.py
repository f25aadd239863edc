"""Seeded synthetic MOREA workloads (SURVEY.md §8(d) "Synthetic inputs").

Input generation only -- no method arithmetic lives here (see package doc).

Geometry convention (reading O1): all positions are in voxel-index
units, voxel (i, j, k) has its centre at (i, j, k); volumes are float32 arrays
of shape (nz, ny, nx), i.e. x-fastest when flattened.  Spacing is isotropic
1.5 mm as in the paper (§5.1, "resampled to (1.5,1.5,1.5)mm").

Configs (BASELINE.json `configs`):
  C1 16^3 ball, Kuhn 3x3x3 lattice (48 tets), P = 8,  K = 1
  C2 64^3 phantom, jittered Kuhn 5x5x6 lattice (480 tets), P = 64, K = 4
  C3 128^3 phantom, Delaunay of 600 points, P = 256, K = 7
  C4 256x256x96 phantom, Delaunay of 600 points, P = 512, K = 7
  C5 = C4 with P = 4096 (sharded over GPUs)
Seeds: phantom 17, mesh 23, population 29, FOS 31, each + 1000 * config index.
"""
from __future__ import annotations

import dataclasses
import numpy as np

SPACING_MM = 1.5
SEVEN = ["bladder", "bones", "rectum", "anal_canal", "sigmoid", "bowel", "body"]

CONFIGS = {
    1: dict(name="C1", dims=(16, 16, 16), mesh="kuhn_c1", P=8, pairs=["ball"]),
    2: dict(name="C2", dims=(64, 64, 64), mesh="kuhn_c2", P=64,
            pairs=["bladder", "bones", "bowel", "body"]),
    3: dict(name="C3", dims=(128, 128, 128), mesh="delaunay", P=256, pairs=SEVEN),
    4: dict(name="C4", dims=(256, 256, 96), mesh="delaunay", P=512, pairs=SEVEN),
    5: dict(name="C5", dims=(256, 256, 96), mesh="delaunay", P=4096, pairs=SEVEN),
}


@dataclasses.dataclass
class Workload:
    name: str
    dims: tuple            # (nx, ny, nz)
    spacing: np.ndarray    # (3,) float64 mm
    I_s: np.ndarray        # (nz, ny, nx) float32, >= 0, background exactly 0
    I_t: np.ndarray
    pairs: list
    cs_off: np.ndarray     # (K+1,) int64 CSR offsets into cs_xyz
    cs_xyz: np.ndarray     # (Ms, 3) float32 voxel units
    ct_off: np.ndarray
    ct_xyz: np.ndarray
    r_mm: float
    base: np.ndarray       # (N, 3) float32 voxel units
    tets: np.ndarray       # (T, 4) int32
    c_delta: np.ndarray    # (T,) float32
    offsets: np.ndarray    # (P, N, 6) float32: (src dx,dy,dz, tgt dx,dy,dz)
    fixed_axes: np.ndarray  # (N, 3) bool: coordinate pinned to the hull
    seed_index: int = 0

    @property
    def V(self):
        nx, ny, nz = self.dims
        return nx * ny * nz

    @property
    def N(self):
        return self.base.shape[0]

    @property
    def T(self):
        return self.tets.shape[0]

    @property
    def P(self):
        return self.offsets.shape[0]


# ----------------------------------------------------------------------------
# Phantom
# ----------------------------------------------------------------------------

def _grid(dims):
    nx, ny, nz = dims
    z, y, x = np.meshgrid(np.arange(nz, dtype=np.float64), np.arange(ny, dtype=np.float64),
                          np.arange(nx, dtype=np.float64), indexing="ij")
    return np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)


class Phantom:
    """Analytic CT-shaped phantom in [0, 1], air exactly 0.0."""

    def __init__(self, dims, kind, rng):
        self.dims = np.asarray(dims, dtype=np.float64)
        self.kind = kind
        self.c = (self.dims - 1.0) / 2.0
        self.h = self.dims / 2.0
        n_min = float(self.dims.min())
        if kind == "ball":
            self.bladder_c = self.c.copy()
            self.R0 = 0.32 * n_min
        else:
            self.bladder_c = self.c + np.array([0.0, 0.18, 0.05]) * self.h
            self.R0 = 0.16 * n_min
        # three seeded sinusoids of soft-tissue texture
        self.tex_k = rng.normal(size=(3, 3)) * 5.0
        self.tex_ph = rng.uniform(0, 2 * np.pi, size=3)
        # gas pockets inside the bowel, in normalised coordinates
        n_gas = int(rng.integers(3, 7))
        self.gas_c = np.array([-0.05, -0.25, 0.25]) + rng.uniform(-1, 1, size=(n_gas, 3)) * \
            np.array([0.22, 0.1, 0.15])
        self.gas_r = rng.uniform(0.03, 0.06, size=n_gas)

    def _w(self, p):
        return (p - self.c) / self.h

    @staticmethod
    def _ell(w, c, r):
        return (((w[:, 0] - c[0]) / r[0]) ** 2 + ((w[:, 1] - c[1]) / r[1]) ** 2
                + ((w[:, 2] - c[2]) / r[2]) ** 2)

    def masks(self, p):
        """Boolean masks of every object at points p (N x 3 voxel coords)."""
        w = self._w(p)
        m = {}
        rb = np.linalg.norm(p - self.bladder_c, axis=1)
        if self.kind == "ball":
            m["ball"] = rb <= self.R0
            return m
        m["body"] = self._ell(w, (0, 0, 0), (0.88, 0.72, 0.80)) <= 1
        m["bowel"] = self._ell(w, (-0.05, -0.25, 0.25), (0.35, 0.2, 0.3)) <= 1
        m["sigmoid"] = self._ell(w, (0.25, 0.2, 0.45), (0.15, 0.1, 0.15)) <= 1
        m["rectum"] = self._ell(w, (0.0, 0.45, -0.2), (0.12, 0.1, 0.35)) <= 1
        m["anal_canal"] = self._ell(w, (0.0, 0.48, -0.62), (0.07, 0.06, 0.15)) <= 1
        m["bladder"] = rb <= self.R0
        b1 = self._ell(w, (0.55, 0.25, -0.1), (0.15, 0.15, 0.3))
        b2 = self._ell(w, (-0.55, 0.25, -0.1), (0.15, 0.15, 0.3))
        m["bones"] = (b1 <= 1) | (b2 <= 1)
        m["_marrow"] = (b1 <= 0.55) | (b2 <= 0.55)
        gas = np.zeros(len(p), dtype=bool)
        for c, r in zip(self.gas_c, self.gas_r):
            gas |= self._ell(w, c, (r, r * self.h[0] / self.h[1], r * self.h[0] / self.h[2])) <= 1
        m["_gas"] = gas & m["bowel"]
        return m

    def values(self, p, m=None):
        m = self.masks(p) if m is None else m
        w = self._w(p)
        v = np.zeros(len(p), dtype=np.float64)
        if self.kind == "ball":
            tex = np.sin(w @ self.tex_k[0] + self.tex_ph[0])
            v[m["ball"]] = (0.5 + 0.05 * tex)[m["ball"]]
            return v.astype(np.float32)
        tex = sum(np.sin(w @ self.tex_k[i] + self.tex_ph[i]) for i in range(3)) / 3.0
        v[m["body"]] = (0.30 + 0.02 * tex)[m["body"]]
        for name, val in (("bowel", 0.28), ("sigmoid", 0.29), ("rectum", 0.26),
                          ("anal_canal", 0.27), ("bladder", 0.22), ("bones", 0.95),
                          ("_marrow", 0.55)):
            v[m[name]] = val
        v[m["_gas"]] = 0.0
        return v.astype(np.float32)


# ----------------------------------------------------------------------------
# Known warp phi = S o R: radial shrink R of the bladder (R1 = 0.7 R0, C^1
# falloff to identity at 2 R0) followed by a smooth global field S(y) = y + v(y).
# ----------------------------------------------------------------------------

class Warp:
    def __init__(self, phantom: Phantom, rng, amplitude=None):
        self.c_b = phantom.bladder_c
        self.R0 = phantom.R0
        dims = phantom.dims
        self.dims = dims
        self.A = float(min(1.5, 0.02 * dims.min())) if amplitude is None else amplitude
        self.ph = rng.uniform(0, 2 * np.pi, size=3)

    def _g(self, r):
        """Inward radial displacement: 0.3 r inside R0, cubic C^1 falloff to 0 at 2 R0."""
        R0 = self.R0
        t = (r - R0) / R0
        out = np.where(r <= R0, 0.3 * r, 0.3 * R0 * (1 + t - 5 * t * t + 3 * t ** 3))
        return np.where(r >= 2 * R0, 0.0, out)

    def _s(self, r):
        return r - self._g(r)

    def radial(self, p):
        d = p - self.c_b
        r = np.linalg.norm(d, axis=1)
        scale = np.where(r > 0, self._s(r) / np.where(r > 0, r, 1.0), 1.0)
        return self.c_b + d * scale[:, None]

    def radial_inv(self, y):
        d = y - self.c_b
        rho = np.linalg.norm(d, axis=1)
        r = rho.copy()
        inside = rho < 2 * self.R0
        if inside.any():
            lo = np.zeros(inside.sum())
            hi = np.full(inside.sum(), 2 * self.R0)
            target = rho[inside]
            for _ in range(60):
                mid = 0.5 * (lo + hi)
                below = self._s(mid) < target
                lo = np.where(below, mid, lo)
                hi = np.where(below, hi, mid)
            r[inside] = 0.5 * (lo + hi)
        scale = np.where(rho > 0, r / np.where(rho > 0, rho, 1.0), 1.0)
        return self.c_b + d * scale[:, None]

    def v(self, y):
        n = self.dims
        return self.A * np.stack([
            np.sin(2 * np.pi * (y[:, 1] + 0.5) / n[1] + self.ph[0]),
            np.sin(2 * np.pi * (y[:, 2] + 0.5) / n[2] + self.ph[1]),
            np.sin(2 * np.pi * (y[:, 0] + 0.5) / n[0] + self.ph[2])], axis=1)

    def forward(self, p):
        y = self.radial(p)
        return y + self.v(y)

    def inverse(self, x):
        y = x.copy()
        for _ in range(12):   # contraction factor A*2*pi/n <= 0.13
            y = x - self.v(y)
        return self.radial_inv(y)


# ----------------------------------------------------------------------------
# Contours
# ----------------------------------------------------------------------------

def _fps(points, k, rng):
    """Greedy farthest-point subset of at most k points (seeded start)."""
    if len(points) <= k:
        return points
    if len(points) > 8 * k:
        points = points[rng.choice(len(points), 8 * k, replace=False)]
    sel = [int(rng.integers(len(points)))]
    dist = np.linalg.norm(points - points[sel[0]], axis=1)
    for _ in range(k - 1):
        i = int(np.argmax(dist))
        sel.append(i)
        dist = np.minimum(dist, np.linalg.norm(points - points[i], axis=1))
    return points[np.array(sel)]


def _surface_points(mask3d):
    """Voxel centres of the object that have a 6-neighbour outside it (or the border)."""
    m = mask3d
    inner = m.copy()
    for ax in range(3):
        for sh in (1, -1):
            nb = np.roll(m, sh, axis=ax)
            # voxels at the image border count as surface
            idx = [slice(None)] * 3
            idx[ax] = 0 if sh == 1 else -1
            nb[tuple(idx)] = False
            inner &= nb
    surf = m & ~inner
    z, y, x = np.nonzero(surf)
    return np.stack([x, y, z], axis=1).astype(np.float64)


# ----------------------------------------------------------------------------
# Meshes
# ----------------------------------------------------------------------------

# Kuhn split of a unit cube: 6 tets along the (0,0,0)-(1,1,1) diagonal,
# one per axis permutation.  Conforming across neighbouring cubes.
_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def kuhn_lattice_mesh(xs, ys, zs):
    xs, ys, zs = (np.asarray(a, dtype=np.float64) for a in (xs, ys, zs))
    nx, ny, nz = len(xs), len(ys), len(zs)
    Z, Y, X = np.meshgrid(zs, ys, xs, indexing="ij")
    pts = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)

    def pid(i, j, k):
        return (k * ny + j) * nx + i

    tets = []
    for k in range(nz - 1):
        for j in range(ny - 1):
            for i in range(nx - 1):
                for perm in _PERMS:
                    c = [i, j, k]
                    v = [pid(*c)]
                    for ax in perm:
                        c[ax] += 1
                        v.append(pid(*c))
                    tets.append(v)
    return pts, np.asarray(tets, dtype=np.int32)


def _delaunay_mesh(dims, contour_pts, rng, n_points=600):
    from scipy.spatial import Delaunay
    from scipy.stats import qmc
    n = np.asarray(dims, dtype=np.float64)
    corners = np.array([[x, y, z] for z in (-0.5, n[2] - 0.5) for y in (-0.5, n[1] - 0.5)
                        for x in (-0.5, n[0] - 0.5)])
    n_free = n_points - 8
    n_sobol = int(round(0.1 * n_free))
    n_contour = n_free - n_sobol
    cpts = _fps(contour_pts, n_contour, rng)
    sob = qmc.Sobol(d=3, scramble=True, seed=int(rng.integers(2**31))).random(n_sobol)
    sob = 2.0 + sob * (n - 5.0)
    pts = np.vstack([corners, cpts, sob])
    tri = Delaunay(pts)
    return pts, tri.simplices.astype(np.int32)


def _fixed_axes(pts, dims):
    n = np.asarray(dims, dtype=np.float64)
    return (pts <= -0.5) | (pts >= n - 0.5)


def _min_incident_altitude(pts, tets):
    """Shortest vertex-to-opposite-face distance over each point's incident tets.

    Used only to scale the population noise so that most solutions are
    fold-free (slivers get proportionally less motion); it decides nothing the
    evaluator outputs.
    """
    N = len(pts)
    best = np.full(N, np.inf)
    P = pts[tets]  # (T, 4, 3)
    vol6 = np.abs(np.einsum("ij,ij->i", np.cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0]),
                            P[:, 3] - P[:, 0]))
    alt = np.full(len(tets), np.inf)
    for k in range(4):
        f = [j for j in range(4) if j != k]
        area2 = np.linalg.norm(np.cross(P[:, f[1]] - P[:, f[0]], P[:, f[2]] - P[:, f[0]]), axis=1)
        alt = np.minimum(alt, vol6 / np.maximum(area2, 1e-300))
    for k in range(4):
        np.minimum.at(best, tets[:, k], alt)
    return best


# ----------------------------------------------------------------------------
# Workload assembly
# ----------------------------------------------------------------------------

def make_workload(cfg_index: int, P: int | None = None, with_fold_solutions: bool = True) -> Workload:
    spec = CONFIGS[cfg_index]
    dims = spec["dims"]
    rng_ph = np.random.default_rng(17 + 1000 * cfg_index)
    rng_mesh = np.random.default_rng(23 + 1000 * cfg_index)
    rng_pop = np.random.default_rng(29 + 1000 * cfg_index)
    P = spec["P"] if P is None else P

    phantom = Phantom(dims, "ball" if spec["mesh"] == "kuhn_c1" else "ct", rng_ph)
    warp = Warp(phantom, rng_ph)
    grid = _grid(dims)
    nx, ny, nz = dims
    masks = phantom.masks(grid)
    I_s = phantom.values(grid, masks).reshape(nz, ny, nx)
    I_t = phantom.values(warp.inverse(grid)).reshape(nz, ny, nx)

    # contours: surface voxel centres of each source object, jittered, thinned
    cs, ct = [], []
    for name in spec["pairs"]:
        surf = _surface_points(masks[name].reshape(nz, ny, nx))
        surf = surf + rng_ph.uniform(-0.25, 0.25, size=surf.shape)
        surf = _fps(surf, 2000, rng_ph)
        cs.append(surf.astype(np.float32))
        ct.append(warp.forward(surf.astype(np.float64)).astype(np.float32))
    cs_off = np.concatenate([[0], np.cumsum([len(c) for c in cs])]).astype(np.int64)
    ct_off = np.concatenate([[0], np.cumsum([len(c) for c in ct])]).astype(np.int64)

    # mesh
    n = np.asarray(dims, dtype=np.float64)
    if spec["mesh"] == "kuhn_c1":
        xs = [-0.5, (n[0] - 1) / 2, n[0] - 0.5]
        base, tets = kuhn_lattice_mesh(xs, [-0.5, (n[1] - 1) / 2, n[1] - 0.5],
                                       [-0.5, (n[2] - 1) / 2, n[2] - 0.5])
    elif spec["mesh"] == "kuhn_c2":
        base, tets = kuhn_lattice_mesh(np.linspace(-0.5, n[0] - 0.5, 5),
                                       np.linspace(-0.5, n[1] - 0.5, 5),
                                       np.linspace(-0.5, n[2] - 0.5, 6))
        cell = np.array([(n[0]) / 4, (n[1]) / 4, (n[2]) / 5])
        fixed = _fixed_axes(base, dims)
        jit = rng_mesh.uniform(-0.2, 0.2, size=base.shape) * cell
        base = base + np.where(fixed, 0.0, jit)
    else:
        allc = np.vstack(cs).astype(np.float64)
        base, tets = _delaunay_mesh(dims, allc, rng_mesh)
    base = base.astype(np.float32)
    fixed = _fixed_axes(base.astype(np.float64), dims)
    T = len(tets)
    c_delta = np.ones(T, dtype=np.float32)

    offsets = make_population(base, tets, fixed, warp, P, rng_pop, with_fold_solutions)
    r_mm = 0.025 * dims[0] * SPACING_MM
    return Workload(name=spec["name"], dims=tuple(dims), spacing=np.full(3, SPACING_MM),
                    I_s=I_s, I_t=I_t, pairs=list(spec["pairs"]), cs_off=cs_off,
                    cs_xyz=np.vstack(cs).astype(np.float32), ct_off=ct_off,
                    ct_xyz=np.vstack(ct).astype(np.float32), r_mm=r_mm, base=base,
                    tets=tets.astype(np.int32), c_delta=c_delta, offsets=offsets,
                    fixed_axes=fixed, seed_index=cfg_index)


def make_population(base, tets, fixed, warp, P, rng, with_fold_solutions=True):
    """Population of dual-mesh offsets (SURVEY.md §8(d) "Population").

    Solution k: O_t = alpha_k (phi(B) - B) + xi, O_s = zeta, alpha_k = k/(P-1);
    noise sigma = min(0.3, 0.08 * smallest incident altitude) voxels; pinned hull
    coordinates get no motion.  Solution 0 is the identity.  Solutions
    k = 7 (mod 16) get one interior vertex reflected through the centroid of the
    opposite face of an incident tet (target side), i.e. pushed across it.
    """
    B = base.astype(np.float64)
    N = len(B)
    free = ~fixed
    sigma = np.minimum(0.3, 0.08 * _min_incident_altitude(B, tets))[:, None]
    disp = warp.forward(B) - B
    out = np.zeros((P, N, 6), dtype=np.float64)
    interior = np.nonzero(~fixed.any(axis=1))[0]
    for k in range(1, P):
        alpha = k / max(P - 1, 1)
        zeta = rng.normal(size=(N, 3)) * sigma
        xi = rng.normal(size=(N, 3)) * sigma
        out[k, :, 0:3] = np.where(free, zeta, 0.0)
        out[k, :, 3:6] = np.where(free, alpha * disp + xi, 0.0)
        if with_fold_solutions and k % 16 == 7 and len(interior):
            j = int(interior[rng.integers(len(interior))])
            inc = np.nonzero((tets == j).any(axis=1))[0]
            t = tets[inc[rng.integers(len(inc))]]
            others = [v for v in t if v != j]
            Xt = B + out[k, :, 3:6]
            c = Xt[others].mean(axis=0)
            out[k, j, 3:6] = (2 * c - Xt[j]) - B[j]
    return out.astype(np.float32)


# ----------------------------------------------------------------------------
# FOS linkage (bench-side; §4.2.1)
# ----------------------------------------------------------------------------

def fos_plan(tets, N, seed=0):
    """Edges -> greedy set cover -> interaction graph -> DSATUR colour classes.

    Tie rules: set cover picks the edge covering the most
    uncovered points, ties by lowest edge id; DSATUR picks max saturation, then
    max degree, then lowest id.  Returns dict(edges=(E,2), colours=(E,),
    classes=list of arrays of element ids, incident=list of tet arrays per point).
    """
    tets = np.asarray(tets)
    pairs = set()
    for a in range(4):
        for b in range(a + 1, 4):
            lo = np.minimum(tets[:, a], tets[:, b])
            hi = np.maximum(tets[:, a], tets[:, b])
            pairs.update(zip(lo.tolist(), hi.tolist()))
    edges = np.array(sorted(pairs), dtype=np.int64)
    covered = np.zeros(N, dtype=bool)
    chosen = []
    while not covered.all():
        gain = (~covered[edges[:, 0]]).astype(int) + (~covered[edges[:, 1]]).astype(int)
        e = int(np.argmax(gain))
        if gain[e] == 0:
            raise ValueError("isolated point")
        chosen.append(e)
        covered[edges[e]] = True
    elems = edges[np.array(chosen)]
    incident = [[] for _ in range(N)]
    for t, tv in enumerate(tets.tolist()):
        for v in tv:
            incident[v].append(t)
    incident = [np.array(sorted(set(x)), dtype=np.int64) for x in incident]
    deps = [np.union1d(incident[a], incident[b]) for a, b in elems.tolist()]
    E = len(elems)
    owner = {}
    for i, d in enumerate(deps):
        for t in d.tolist():
            owner.setdefault(t, []).append(i)
    adj = [set() for _ in range(E)]
    for lst in owner.values():
        for i in lst:
            adj[i].update(lst)
    for i in range(E):
        adj[i].discard(i)
    colours = np.full(E, -1, dtype=np.int64)
    sat = [set() for _ in range(E)]
    deg = np.array([len(a) for a in adj])
    for _ in range(E):
        best, key = -1, None
        for i in range(E):
            if colours[i] >= 0:
                continue
            k = (len(sat[i]), deg[i], -i)
            if key is None or k > key:
                best, key = i, k
        c = 0
        while c in sat[best]:
            c += 1
        colours[best] = c
        for j in adj[best]:
            sat[j].add(c)
    classes = [np.nonzero(colours == c)[0] for c in range(colours.max() + 1)]
    return dict(edges=elems, colours=colours, classes=classes, incident=incident, deps=deps)


def partial_request(w: Workload, plan, kind="class", class_index=0, seed=31, sigma=0.5):
    """Build a multi-group partial-evaluation request (SURVEY.md §8(d) partial sweep).

    kind: "class" (each element of one colour class is a group of 2 points),
    "edges4"/"edges16" (groups of 4/16 edges of one colour class), "wholeclass"
    (one group with every point of the colour class), "all" (one group with
    every point).  New values = base offsets + N(0, sigma^2) on all
    6 coordinates (pinned hull coordinates unchanged).
    Returns (grp_off int32 (G+1,), changed_pts int32 (S,), new_vals float32 (P, S, 6)).
    """
    rng = np.random.default_rng(seed + 1000 * w.seed_index)
    if kind == "all":
        groups = [np.arange(w.N)]
    else:
        cls = plan["classes"][class_index % len(plan["classes"])]
        elems = plan["edges"][cls]
        per = {"class": 1, "edges4": 4, "edges16": 16, "wholeclass": len(elems)}[kind]
        groups = []
        for i in range(0, len(elems), per):
            groups.append(np.unique(elems[i:i + per].ravel()))
    grp_off = np.concatenate([[0], np.cumsum([len(g) for g in groups])]).astype(np.int32)
    changed = np.concatenate(groups).astype(np.int32)
    fixed6 = np.concatenate([w.fixed_axes, w.fixed_axes], axis=1)[changed]  # (S, 6)
    noise = rng.normal(size=(w.P, len(changed), 6)) * sigma
    new_vals = w.offsets[:, changed, :].astype(np.float64) + np.where(fixed6[None], 0.0, noise)
    return grp_off, changed, np.ascontiguousarray(new_vals, dtype=np.float32)


def random_tiny_mesh(dims, n_inner, seed):
    """Small Delaunay mesh over the image extent (hull at -0.5, n-0.5) for pin tests."""
    from scipy.spatial import Delaunay
    rng = np.random.default_rng(seed)
    n = np.asarray(dims, dtype=np.float64)
    corners = np.array([[x, y, z] for z in (-0.5, n[2] - 0.5) for y in (-0.5, n[1] - 0.5)
                        for x in (-0.5, n[0] - 0.5)])
    inner = 0.3 + rng.uniform(size=(n_inner, 3)) * (n - 1.6)
    pts = np.vstack([corners, inner])
    return pts.astype(np.float32), Delaunay(pts).simplices.astype(np.int32)

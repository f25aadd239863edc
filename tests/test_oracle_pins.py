"""Pins of the CPU oracle against things other than itself (run with -m "not gpu").

Every pin is a value the paper prints, a closed form, a textbook/library routine
(scipy), an exact brute force with a different algorithm (Python Fractions), or
an invariant the method guarantees.  Citations: PAPER.md line numbers (L…),
SPEC.md (S:L…), readings O1..O13.
"""
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O
from synth import kuhn_lattice_mesh, random_tiny_mesh
from tests.helpers import FracTet, axis_set_frac, blob_volume, frac_det, make_oracle, q10

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append([float(v) for v in line.split()])
    return rows


# --------------------------------------------------------------------------- h, det, canon
def test_h_golden():
    """h of §4.1.2 (L318-322); values from SPEC S:L416."""
    for a, b, fg, exp in _golden("h_values.txt"):
        assert O.h(a, b, int(fg)) == pytest.approx(exp, abs=1e-15)


def test_signed_volume_golden():
    """Signed volume (App. A.4); SPEC S:L145-147 examples."""
    for row in _golden("signed_volume.txt"):
        Q = (np.array(row[:12]) * 1024).astype(np.int64).reshape(4, 3)
        s, det = O.signed_det(Q)
        assert det / (6 * 1024 ** 3) == pytest.approx(row[12], abs=1e-15)
        assert s == int(np.sign(row[12]))


def test_signed_det_exact_vs_fraction_elimination():
    """Exact int128 determinant vs fraction-free elimination on +-2^20 inputs (bound of O1)."""
    rng = np.random.default_rng(5)
    for _ in range(300):
        Q = rng.integers(-(2 ** 19), 2 ** 19, size=(4, 3))
        if rng.uniform() < 0.2:  # force coplanar / repeated cases
            Q[3] = Q[0] + (Q[1] - Q[0]) * rng.integers(-2, 3) + (Q[2] - Q[0]) * rng.integers(-2, 3)
        s, det = O.signed_det(Q)
        E = [[int(Q[k + 1][a] - Q[0][a]) for k in range(3)] for a in range(3)]
        ref = frac_det(E)
        assert det == ref
        assert s == (ref > 0) - (ref < 0)


def test_canon_round_half_even():
    """O1: Q = round-half-even(1024 B + 1024 O) in fp64 (ties to even)."""
    cases = [(0.0, 0.5 / 1024), (0.0, 1.5 / 1024), (0.0, -0.5 / 1024), (3.25, 2.5 / 1024),
             (-0.5, 0.1234567), (255.5, -1e-4), (17.0, 1.0 / 3.0)]
    for b, o in cases:
        assert O.canon(b, o) == q10(b, o)
    assert O.canon(0.0, 0.5 / 1024) == 0 and O.canon(0.0, 1.5 / 1024) == 2


# --------------------------------------------------------------------------- trilinear
def test_trilinear_golden():
    """App. A.2 L744 interpolation; SPEC S:L59-61 (centre, midpoint 2,4 -> 3, clamp)."""
    vol = np.array([2, 4, 2, 4, 2, 4, 2, 4], dtype=np.float32).reshape(2, 2, 2)
    for x, y, z, exp in _golden("trilinear.txt"):
        assert O.trilinear(vol, (x, y, z)) == pytest.approx(exp, abs=1e-14)


def test_trilinear_vs_scipy_map_coordinates():
    """O5 pinned to scipy.ndimage.map_coordinates(order=1, mode='nearest')."""
    from scipy.ndimage import map_coordinates
    rng = np.random.default_rng(3)
    vol = rng.uniform(0, 1, size=(7, 9, 11)).astype(np.float32)
    pts = rng.uniform(-2.0, 12.0, size=(400, 3))
    pts[:50] = np.round(pts[:50])  # lattice points incl. outside
    ref = map_coordinates(vol.astype(np.float64), pts[:, ::-1].T, order=1, mode="nearest")
    got = np.array([O.trilinear(vol, p) for p in pts])
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)


def test_trilinear_reproduces_affine():
    """A volume affine in position is reproduced exactly inside."""
    nz, ny, nx = 6, 7, 8
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    vol = (0.5 + 0.25 * x + 0.125 * y - 0.0625 * z).astype(np.float32)
    rng = np.random.default_rng(4)
    for p in rng.uniform(0, [nx - 1, ny - 1, nz - 1], size=(100, 3)):
        assert O.trilinear(vol, p) == pytest.approx(0.5 + 0.25 * p[0] + 0.125 * p[1] - 0.0625 * p[2],
                                                    abs=1e-12)


# --------------------------------------------------------------------------- ownership (O3)
def _frac_owner_map(orc, base, tets, off, side, dims):
    """Per-voxel x all-tets exact brute force with Fraction barycentrics."""
    nx, ny, nz = dims
    Qall = np.array([[q10(base[j, a], off[j, 3 * side + a]) for a in range(3)] for j in range(len(base))])
    fts = [FracTet(Qall[t]) for t in tets]
    owner = np.full(nx * ny * nz, -1, dtype=np.int32)
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                hits = [t for t, ft in enumerate(fts) if ft.owns((x, y, z))]
                owner[(z * ny + y) * nx + x] = -1 if not hits else (hits[0] if len(hits) == 1 else -2)
    return owner


@pytest.mark.parametrize("seed", [1, 2])
def test_ownership_vs_fraction_bruteforce_random_mesh(seed):
    """O3 owner map == per-voxel x all-tets exact brute force (8^3), random Delaunay + offsets."""
    dims = (8, 8, 8)
    base, tets = random_tiny_mesh(dims, 10, seed)
    rng = np.random.default_rng(seed)
    off = np.zeros((len(base), 6), np.float32)
    off[8:] = rng.normal(0, 0.15, size=(len(base) - 8, 6))
    I = blob_volume(dims, seed)
    orc = make_oracle(dims, I, I, base, tets)
    for side in (0, 1):
        got = orc.owner_map(off, side)
        ref = _frac_owner_map(orc, base, tets, off, side, dims)
        np.testing.assert_array_equal(got, ref)


def test_ownership_tie_heavy_integer_kuhn_exactly_once():
    """Integer-vertex Kuhn mesh: faces, edges, vertices and hull faces hit voxel centres.

    Every lattice point q with q + (e, e^2, e^3) inside the hull [0, L]^3 has
    exactly one owner, every other point none (O3 'consequence at the hull').
    Also checked against the Fraction brute force on the full 9^3 grid.
    """
    L = 8
    dims = (10, 10, 10)
    base, tets = kuhn_lattice_mesh([0, 4, 8], [0, 4, 8], [0, 4, 8])
    base = base.astype(np.float32)
    I = blob_volume(dims, 7)
    orc = make_oracle(dims, I, I, base, tets)
    off = np.zeros((len(base), 6), np.float32)
    own = orc.owner_map(off, 0).reshape(10, 10, 10)
    z, y, x = np.meshgrid(range(10), range(10), range(10), indexing="ij")
    inside = (x < L) & (y < L) & (z < L)
    assert (own[inside] >= 0).all()
    assert (own[~inside] == -1).all()
    ref = _frac_owner_map(orc, base, tets, off, 0, dims)
    np.testing.assert_array_equal(own.ravel(), ref)


def test_ownership_partition_bench_hull(wl):
    """Hull at the image extent (-0.5, n-0.5): every voxel owned exactly once when unfolded."""
    for idx in (1, 2):
        w = wl(idx)
        orc = O.Oracle.from_workload(w)
        for k in (0, 1, 2):
            assert orc.check_folds(w.offsets[k])[0] == 0
            for side in (0, 1):
                own = orc.owner_map(w.offsets[k], side)
                assert (own >= 0).all(), (idx, k, side)
            _, acc = orc.eval(w.offsets[k])
            assert acc.n_samples == 2 * w.V


# --------------------------------------------------------------------------- transform (O4), exact split (O6)
def _affine_problem(n=12, A=None, b=None, seed=0):
    """Half-integer Kuhn lattice over the image; target = A source + b exactly in Q.10."""
    g = [-0.5, 3.5, 7.5, n - 0.5]
    base, tets = kuhn_lattice_mesh(g, g, g)
    base = base.astype(np.float32)
    if A is None:
        A = np.eye(3) + np.array([[17, 5, -7], [-3, 11, 6], [4, -9, 13]]) / 256.0
    if b is None:
        b = np.array([0.3291015625, -0.4052734375, 0.2177734375])  # odd multiples of 1/1024
    Xt = base.astype(np.float64) @ A.T + b
    off = np.zeros((len(base), 6), np.float32)
    off[:, 3:] = (Xt - base).astype(np.float32)
    assert np.array_equal(off[:, 3:].astype(np.float64) + base, Xt)  # exact in fp32
    return (n, n, n), base, tets, off, A, b


def test_transform_identity_and_translation_exact():
    """O4 displacement form: identity -> x = q exactly; translation t -> q + t exactly."""
    dims = (10, 10, 10)
    base, tets = random_tiny_mesh(dims, 8, 11)
    I = blob_volume(dims, 3)
    orc = make_oracle(dims, I, I, base, tets)
    t = np.array([1.25, -0.5, 2.0009765625], np.float32)  # Q.10-exact
    for shift in (np.zeros(3, np.float32), t):
        off = np.zeros((len(base), 6), np.float32)
        off[:, 3:] = shift
        rng = np.random.default_rng(1)
        n_owned = 0
        for _ in range(200):
            q = rng.integers(0, 10, size=3)
            for tt in range(len(tets)):
                r = orc.sample_debug(off, tt, 0, q)
                if r["owned"]:
                    n_owned += 1
                    assert np.array_equal(r["x"], q + shift.astype(np.float64))
        assert n_owned == 200


def test_transform_global_affine_and_exact_sets_vs_fraction():
    """Piecewise-linear map reproduces a global affine map; exact floor/integer decisions.

    Pins O4 (x = A q + b for every owned q, fp64 within 1e-12) and the exact
    contributing index sets of O6 against Fraction arithmetic.
    """
    dims, base, tets, off, A, b = _affine_problem()
    I = blob_volume(dims, 5)
    orc = make_oracle(dims, I, I, base, tets)
    rng = np.random.default_rng(2)
    Af = [[Fraction(v).limit_denominator(1 << 12) for v in row] for row in A]
    bf = [Fraction(v).limit_denominator(1 << 12) for v in b]
    checked = 0
    for _ in range(120):
        q = rng.integers(0, dims[0], size=3)
        for tt in range(len(tets)):
            r = orc.sample_debug(off, tt, 0, q)
            if not r["owned"]:
                continue
            xf = [sum(Af[i][j] * int(q[j]) for j in range(3)) + bf[i] for i in range(3)]
            np.testing.assert_allclose(r["x"], [float(v) for v in xf], rtol=0, atol=1e-12)
            for a in range(3):
                s = axis_set_frac(xf[a], dims[a])
                got = [int(v) for v in r["sets"][a, 1:1 + r["sets"][a, 0]]]
                assert got == s
            checked += 1
    assert checked == 120


def test_transform_barycentric_fraction_random_mesh():
    """O4 on random meshes: x = sum_k lambda_k X'_k with Fraction barycentrics; sets exact."""
    dims = (9, 9, 9)
    base, tets = random_tiny_mesh(dims, 9, 21)
    rng = np.random.default_rng(21)
    off = np.zeros((len(base), 6), np.float32)
    off[8:] = rng.normal(0, 0.2, size=(len(base) - 8, 6))
    I = blob_volume(dims, 9)
    orc = make_oracle(dims, I, I, base, tets)
    Q = [np.array([[q10(base[j, a], off[j, 3 * s + a]) for a in range(3)] for j in range(len(base))])
         for s in (0, 1)]
    checked = 0
    for tt in range(len(tets)):
        for side in (0, 1):
            ft = FracTet(Q[side][tets[tt]])
            cen = np.array(ft.Qv).mean(0) / 1024.0
            for _ in range(6):
                q = np.clip(np.round(cen + rng.normal(0, 1.0, 3)), 0, 8).astype(np.int64)
                r = orc.sample_debug(off, tt, side, q)
                if not ft.owns(q):
                    assert not r["owned"]
                    continue
                assert r["owned"]
                lam, _ = ft.bary([1024 * int(c) for c in q])
                Xo = Q[1 - side][tets[tt]]
                xf = [sum(lam[k] * int(Xo[k][a]) for k in range(4)) / 1024 for a in range(3)]
                np.testing.assert_allclose(r["x"], [float(v) for v in xf], rtol=0, atol=1e-11)
                for a in range(3):
                    got = [int(v) for v in r["sets"][a, 1:1 + r["sets"][a, 0]]]
                    assert got == axis_set_frac(xf[a], dims[a])
                checked += 1
    assert checked > 20


def test_exact_split_on_integer_landing_positions():
    """Positions landing exactly on lattice planes (x = 2 q - c) take the exact single-corner set."""
    n = 12
    A = 2.0 * np.eye(3)
    b = np.array([-5.5, -5.5, -5.5])  # x = 2 q - 5.5 + ... lands on half-integers? use integer b
    b = np.array([-6.0, -5.0, -4.0])
    dims, base, tets, off, A, b = _affine_problem(n, A=A, b=b)
    I = blob_volume(dims, 13, frac_zero=0.5)
    orc = make_oracle(dims, I, I, base, tets)
    for q in [(3, 4, 5), (5, 5, 5), (6, 2, 7), (1, 1, 1), (10, 10, 10)]:
        for tt in range(len(tets)):
            r = orc.sample_debug(off, tt, 0, np.array(q))
            if r["owned"]:
                x = 2 * np.array(q) + b
                exp = [int(min(max(v, 0), n - 1)) for v in x]
                assert [int(r["sets"][a, 0]) for a in range(3)] == [1, 1, 1]
                assert [int(r["sets"][a, 1]) for a in range(3)] == exp
                assert r["fg"] == (I[exp[2], exp[1], exp[0]] > 0)
                assert r["b"] == pytest.approx(float(I[exp[2], exp[1], exp[0]]), abs=1e-12)


# --------------------------------------------------------------------------- f_intensity closed forms (O6/O7)
def _h_vec(a, b):
    """h of L318-322 on arrays where the footprint case is read from b > 0 (generic positions)."""
    return np.where((a > 0) & (b > 0), (a - b) ** 2, np.where((a == 0) & (b == 0), 0.0, 1.0))


def test_f_int_identity_is_voxelwise_h(wl):
    """north_star: 'the identity deformation gives SSD(source, target)' -> sum_v h(I_s, I_t) / V."""
    for idx in (1, 2):
        w = wl(idx)
        orc = O.Oracle.from_workload(w)
        obj, acc = orc.eval(w.offsets[0])
        a = w.I_s.astype(np.float64).ravel()
        b = w.I_t.astype(np.float64).ravel()
        ref = (_h_vec(a, b).sum() + _h_vec(b, a).sum()) / (2 * w.V)
        assert obj[1] == pytest.approx(ref, rel=1e-12)
        assert obj[0] == 0.0


def test_f_int_global_affine_closed_form():
    """f_int under an exact global affine map == mesh-free map_coordinates evaluation (1e-12)."""
    from scipy.ndimage import map_coordinates
    dims, base, tets, off, A, b = _affine_problem()
    n = dims[0]
    I_s = blob_volume(dims, 31, frac_zero=0.3)
    I_t = blob_volume(dims, 32, frac_zero=0.3)
    orc = make_oracle(dims, I_s, I_t, base, tets)
    obj, acc = orc.eval(off)
    z, y, x = np.meshgrid(range(n), range(n), range(n), indexing="ij")
    q = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.float64)
    xs = q @ A.T + b
    bs = map_coordinates(I_t.astype(np.float64), xs[:, ::-1].T, order=1, mode="nearest")
    hs = _h_vec(I_s.astype(np.float64).ravel(), bs)
    # target samples: lattice points strictly inside A * box + b
    y_src = (q - b) @ np.linalg.inv(A).T
    margin = np.minimum(y_src + 0.5, (n - 0.5) - y_src).min(axis=1)
    assert np.abs(margin).min() > 1e-6  # no lattice point on the target hull
    inside = margin > 0
    bt = map_coordinates(I_s.astype(np.float64), y_src[inside][:, ::-1].T, order=1, mode="nearest")
    ht = _h_vec(I_t.astype(np.float64).ravel()[inside], bt)
    ref = (hs.sum() + ht.sum()) / (n ** 3 + inside.sum())
    assert acc.n_samples == n ** 3 + inside.sum()
    assert obj[1] == pytest.approx(ref, rel=1e-12)


def _translation_problem(t=(2, -1, 1), seed=4):
    """Special phantom for the exact-zero pin: support and contours away from the border."""
    n = 16
    dims = (n, n, n)
    rng = np.random.default_rng(seed)
    I_s = np.zeros((n, n, n), np.float32)
    I_s[5:11, 5:11, 5:11] = rng.uniform(0.1, 1.0, size=(6, 6, 6)).astype(np.float32)
    I_s[7, 7, 7] = 0.0  # a gas voxel inside the object
    t = np.array(t)
    I_t = np.zeros_like(I_s)
    I_t[5 + t[2]:11 + t[2], 5 + t[1]:11 + t[1], 5 + t[0]:11 + t[0]] = I_s[5:11, 5:11, 5:11]
    cs = [(np.round(rng.uniform(6, 10, size=(40, 3)) * 64) / 64).astype(np.float32)]
    ct = [(cs[0] + t).astype(np.float32)]
    assert np.array_equal(ct[0].astype(np.float64) - t, cs[0].astype(np.float64))
    base, tets = random_tiny_mesh(dims, 14, seed)
    off = np.zeros((len(base), 6), np.float32)
    off[8:, :3] = np.round(rng.normal(0, 0.05, size=(len(base) - 8, 3)) * 1024) / 1024
    off[:, 3:] = off[:, :3] + t
    return dims, I_s, I_t, cs, ct, base, tets, off


def test_integer_translation_gives_exact_zeros():
    """Target mesh = source mesh + integer t on the special phantom: all objectives exactly 0."""
    dims, I_s, I_t, cs, ct, base, tets, off = _translation_problem()
    orc = make_oracle(dims, I_s, I_t, base, tets, cs=cs, ct=ct, r_mm=3.0)
    assert orc.check_folds(off)[0] == 0
    obj, acc = orc.eval(off)
    assert acc.n_samples > 0
    assert obj[0] == 0.0 and obj[1] == 0.0 and obj[2] == 0.0
    # the band is not empty (the zero is not vacuous): at identity the guidance is > 0
    # whenever the contours differ, and source samples near contours exist
    off2 = off.copy()
    off2[:, 3:] = off2[:, :3]
    assert orc.eval(off2)[0][2] > 0.0


# --------------------------------------------------------------------------- distance maps + f_guidance (O8)
def test_distance_map_vs_ckdtree():
    """Exact nearest-point distance maps pinned to scipy.spatial.cKDTree (anisotropic spacing)."""
    from scipy.spatial import cKDTree
    dims = (13, 11, 9)
    spacing = (1.5, 0.8, 2.25)
    rng = np.random.default_rng(8)
    cs = [rng.uniform(-1, 12, size=(57, 3)).astype(np.float32), rng.uniform(0, 8, size=(3, 3)).astype(np.float32)]
    ct = [rng.uniform(0, 10, size=(20, 3)).astype(np.float32), np.array([[4.0, 5.0, 6.0]], np.float32)]
    I = blob_volume(dims, 1)
    base, tets = random_tiny_mesh(dims, 5, 3)
    orc = make_oracle(dims, I, I, base, tets, cs=cs, ct=ct, spacing=spacing)
    nx, ny, nz = dims
    z, y, x = np.meshgrid(range(nz), range(ny), range(nx), indexing="ij")
    q = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.float64)
    for s, cc in ((0, cs), (1, ct)):
        for i, pts in enumerate(cc):
            tree = cKDTree(pts.astype(np.float64) * spacing)
            d, _ = tree.query(q * spacing)
            got = orc.distance_map(s, i)
            np.testing.assert_allclose(got, d.astype(np.float32), rtol=2e-7, atol=0)
    # single point -> Euclidean distance
    d1 = orc.distance_map(1, 1)
    ref = np.sqrt((((q - [4, 5, 6]) * spacing) ** 2).sum(1))
    np.testing.assert_allclose(d1, ref.astype(np.float32), rtol=2e-7)


def test_f_guid_identity_closed_form(wl):
    """At identity: sum_i sum_side w_i sum_{D_i(v) < r} ((r-D)/r)(D_i(v) - D'_i(v))^2 / (2V)."""
    from scipy.spatial import cKDTree
    w = wl(2)
    orc = O.Oracle.from_workload(w)
    obj, acc = orc.eval(w.offsets[0])
    nx, ny, nz = w.dims
    z, y, x = np.meshgrid(range(nz), range(ny), range(nx), indexing="ij")
    q = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.float64) * w.spacing
    K = len(w.pairs)
    tot = 0.0
    sides = [(w.cs_off, w.cs_xyz), (w.ct_off, w.ct_xyz)]
    for s in (0, 1):
        off_s, xyz_s = sides[s]
        off_o, xyz_o = sides[1 - s]
        for i in range(K):
            ws = (off_s[i + 1] - off_s[i]) / off_s[-1]
            D = cKDTree(xyz_s[off_s[i]:off_s[i + 1]].astype(np.float64) * w.spacing).query(q)[0]
            D = D.astype(np.float32).astype(np.float64)
            Do = cKDTree(xyz_o[off_o[i]:off_o[i + 1]].astype(np.float64) * w.spacing).query(q)[0]
            Do = Do.astype(np.float32).astype(np.float64)
            band = D < w.r_mm
            tot += ws * (((w.r_mm - D[band]) / w.r_mm) * (D[band] - Do[band]) ** 2).sum()
    assert obj[2] == pytest.approx(tot / (2 * w.V), rel=1e-6)


def _brute_dmap(q_vox, pts, spacing):
    """D(q) = min_c ||(q - c) * spacing|| by brute force over ALL points (SURVEY §8(c) 'Form'):
    per point dx, dy, dz in fp64, ((dx^2 + dy^2) + dz^2), min, sqrt, rounded once to fp32.
    A different algorithm from the oracle's bucket search, the same arithmetic definition."""
    best = np.full(len(q_vox), np.inf)
    c = pts.astype(np.float64)
    for j in range(len(c)):
        dx = (q_vox[:, 0] - c[j, 0]) * spacing[0]
        dy = (q_vox[:, 1] - c[j, 1]) * spacing[1]
        dz = (q_vox[:, 2] - c[j, 2]) * spacing[2]
        best = np.minimum(best, (dx * dx + dy * dy) + dz * dz)
    return np.sqrt(best).astype(np.float32)


def test_f_guid_global_affine_closed_form():
    """f_guidance under an exact global affine target mesh (x = A q + b at NON-lattice positions)
    == a mesh-free evaluation of eq. L338-342 / App. A.3 L793-796 (reading O8): brute-force
    distance maps at the voxel centres, D'_i interpolated with scipy map_coordinates(order=1,
    mode='nearest') at A q + b (side s) and A^-1 (q - b) (side t).  Pins the oracle's
    trilinear_map at fractional positions (a wrong fractional weight fails it)."""
    from scipy.ndimage import map_coordinates
    dims, base, tets, off, A, b = _affine_problem()
    n = dims[0]
    sp = np.array([1.5, 1.5, 1.5])
    rng = np.random.default_rng(41)
    cs = [rng.uniform(1, n - 2, size=(60, 3)).astype(np.float32),
          rng.uniform(2, n - 3, size=(25, 3)).astype(np.float32)]
    ct = [(cs[0].astype(np.float64) @ A.T + b + rng.normal(0, 0.4, size=(60, 3))).astype(np.float32),
          rng.uniform(2, n - 3, size=(31, 3)).astype(np.float32)]
    r_mm = 4.0
    I = blob_volume(dims, 7)
    orc = make_oracle(dims, I, I, base, tets, cs=cs, ct=ct, r_mm=r_mm, spacing=tuple(sp))
    obj, acc = orc.eval(off)
    z, y, x = np.meshgrid(range(n), range(n), range(n), indexing="ij")
    q = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.float64)
    D = {(s, i): _brute_dmap(q, (cs, ct)[s][i], sp).astype(np.float64) for s in (0, 1) for i in range(2)}
    for (s, i), d in D.items():  # the oracle's stored maps are these exact values
        assert np.array_equal(orc.distance_map(s, i), d.astype(np.float32))
    y_src = (q - b) @ np.linalg.inv(A).T
    margin = np.minimum(y_src + 0.5, (n - 0.5) - y_src).min(axis=1)
    assert np.abs(margin).min() > 1e-6
    inside_t = margin > 0
    pos = {0: (np.ones(len(q), bool), q @ A.T + b), 1: (inside_t, y_src)}
    tot = 0.0
    for s in (0, 1):
        owned, xs = pos[s]
        sizes = [len((cs, ct)[s][i]) for i in range(2)]
        for i in range(2):
            w_i = sizes[i] / sum(sizes)  # |C_i^s| / |G_s| (L340)
            d = D[(s, i)][owned]
            grid = D[(1 - s, i)].reshape(n, n, n)
            Dp = map_coordinates(grid, xs[owned][:, ::-1].T, order=1, mode="nearest")
            bnd = d < r_mm  # strict (eq. L341)
            assert bnd.sum() > 20  # the band is populated on both sides
            tot += w_i * (((r_mm - d[bnd]) / r_mm) * (d[bnd] - Dp[bnd]) ** 2).sum()
    n_tot = n ** 3 + inside_t.sum()
    assert acc.n_samples == n_tot
    assert obj[2] == pytest.approx(tot / n_tot, rel=1e-12)


def test_f_guid_truncation_closed_forms():
    """SPEC S:L426-427 and the strict d < r of eq. L341: a source voxel at distance d = 0 whose
    mapped distance is delta contributes w delta^2; a voxel at exactly d = r contributes 0.
    Identity mesh, one source contour point on voxel centre c, one target point at c + (1/2, 0, 0)
    (distance 0.75 mm from its two nearest voxel centres, 1.5 mm spacing)."""
    dims = (8, 8, 8)
    base, tets = kuhn_lattice_mesh([-0.5, 3.5, 7.5], [-0.5, 3.5, 7.5], [-0.5, 3.5, 7.5])
    base = base.astype(np.float32)
    I = blob_volume(dims, 3)
    c = np.array([[3.0, 4.0, 2.0]], np.float32)
    ct = [c + np.array([0.5, 0.0, 0.0], np.float32)]
    off = np.zeros((len(base), 6), np.float32)
    V = 8 ** 3
    # r = 0.6 mm: source band = {c} (d = 0), target band empty (nearest centre at 0.75 mm)
    orc = make_oracle(dims, I, I, base, tets, cs=[c], ct=ct, r_mm=0.6)
    obj, acc = orc.eval(off)
    assert acc.n_samples == 2 * V
    assert acc.g_sum == 0.75 ** 2  # w = 1, (r - 0)/r = 1, (0 - 0.75)^2 exactly
    assert obj[2] == 0.75 ** 2 / (2 * V)
    # r = 0.75 exactly: the two target-side centres at d = 0.75 = r are NOT in the band
    orc = make_oracle(dims, I, I, base, tets, cs=[c], ct=ct, r_mm=0.75)
    assert orc.eval(off)[1].g_sum == 0.75 ** 2
    # r just above 0.75: they enter with weight (r - 0.75)/r and D_s there = 1.5 mm (one voxel from c)
    r = 0.76
    orc = make_oracle(dims, I, I, base, tets, cs=[c], ct=ct, r_mm=r)
    g = orc.eval(off)[1].g_sum
    ref = 0.75 ** 2 + 2 * ((r - 0.75) / r) * (0.75 - 1.5) ** 2
    assert g == pytest.approx(ref, rel=1e-12)


def test_distance_map_bruteforce_c3_sampled(wl):
    """C3 distance maps of the oracle (bucket search) == SURVEY §8(c)'s brute force, bit-exact,
    on 3000 sampled voxels of every pair and side (the bucket search at full config size)."""
    w = wl(3, 4)
    orc = O.Oracle.from_workload(w)
    nx, ny, nz = w.dims
    rng = np.random.default_rng(5)
    v = rng.integers(0, w.V, size=3000)
    q = np.stack([v % nx, (v // nx) % ny, v // (nx * ny)], 1).astype(np.float64)
    sides = [(w.cs_off, w.cs_xyz), (w.ct_off, w.ct_xyz)]
    for s in (0, 1):
        off_s, xyz_s = sides[s]
        for i in range(len(w.pairs)):
            got = orc.distance_at(s, i, q.astype(np.int64))
            ref = _brute_dmap(q, xyz_s[off_s[i]:off_s[i + 1]], w.spacing)
            assert np.array_equal(got, ref), (s, i)


# --------------------------------------------------------------------------- f_magnitude (O9)
def test_f_mag_closed_forms():
    """Identity/translation -> 0; uniform scale alpha -> (1-alpha)^2 sum c sum |e|^2 / (10T);
    doubling c_delta doubles it."""
    dims, base, tets, off, A, b = _affine_problem(A=1.25 * np.eye(3), b=np.zeros(3))
    I = blob_volume(dims, 2)
    rng = np.random.default_rng(0)
    c = rng.uniform(0.5, 2.0, size=len(tets)).astype(np.float32)
    orc = make_oracle(dims, I, I, base, tets, c_delta=c)
    sp = 1.5
    X = base.astype(np.float64)
    tot = 0.0
    for t, tv in enumerate(tets):
        P = X[tv]
        e2 = sum(np.sum(((P[i] - P[j]) * sp) ** 2) for i in range(4) for j in range(i + 1, 4))
        for k in range(4):
            fc = (P.sum(0) - P[k]) / 3.0
            e2 += np.sum(((P[k] - fc) * sp) ** 2)
        tot += c[t] * e2
    obj, _ = orc.eval(off)
    assert obj[0] == pytest.approx((1 - 1.25) ** 2 * tot / (10 * len(tets)), rel=1e-12)
    orc2 = make_oracle(dims, I, I, base, tets, c_delta=2 * c)
    assert orc2.eval(off)[0][0] == pytest.approx(2 * obj[0], rel=1e-14)
    ident = np.zeros_like(off)
    assert orc.eval(ident)[0][0] == 0.0
    trans = np.zeros_like(off)
    trans[:, :3] = [0.25, 0.5, -0.75]
    trans[:, 3:] = [1.5, -2.0, 0.125]
    assert orc.eval(trans)[0][0] == 0.0


def test_f_mag_spoke_modes_single_tet():
    """Single tet, one vertex-vertex edge longer by delta: the 6 vertex edges and
    4 spokes contribute per their definitions; spoke_mode 1 scales spokes by 3/4."""
    dims = (8, 8, 8)
    base = np.array([[-0.5, -0.5, -0.5], [7.5, -0.5, -0.5], [-0.5, 7.5, -0.5], [-0.5, -0.5, 7.5]], np.float32)
    tets = np.array([[0, 1, 2, 3]], np.int32)
    I = blob_volume(dims, 1)
    off = np.zeros((4, 6), np.float32)
    off[1, 3] = 1.0  # vertex 1 moves +1 voxel in x on the target side
    X = base.astype(np.float64)
    Y = X.copy()
    Y[1, 0] += 1.0

    def L(P, i, j):
        return np.linalg.norm((P[i] - P[j]) * 1.5)

    def S(P, k, scale):
        fc = (P.sum(0) - P[k]) / 3.0
        return np.linalg.norm((P[k] - fc) * 1.5) * scale

    for mode, scale in ((0, 1.0), (1, 0.75)):
        orc = make_oracle(dims, I, I, base, tets, spoke_mode=mode)
        m = sum((L(X, i, j) - L(Y, i, j)) ** 2 for i in range(4) for j in range(i + 1, 4))
        m += sum((S(X, k, scale) - S(Y, k, scale)) ** 2 for k in range(4))
        assert orc.eval(off)[0][0] == pytest.approx(m / 10.0, rel=1e-12)


# --------------------------------------------------------------------------- folds (O2)
def test_fold_fig2_construction():
    """Fig. 2 (L347-373): a point moved across its opposite face flips that tet's sign."""
    dims = (12, 12, 12)
    g = [-0.5, 3.5, 7.5, 11.5]
    base, tets = kuhn_lattice_mesh(g, g, g)
    base = base.astype(np.float32)
    I = blob_volume(dims, 1)
    orc = make_oracle(dims, I, I, base, tets)
    j = 1 * 16 + 1 * 4 + 1  # interior lattice point (1,1,1)
    inc = np.nonzero((tets == j).any(1))[0]
    for t in inc[:6]:
        others = [v for v in tets[t] if v != j]
        c = base[others].astype(np.float64).mean(0)
        for side in (0, 1):
            off = np.zeros((len(base), 6), np.float32)
            off[j, 3 * side:3 * side + 3] = (2 * c - base[j]) - base[j]
            cnt, sev, flags = orc.check_folds(off)
            assert flags[side, t] == 1
            assert flags[1 - side].sum() == 0
            assert cnt == flags.sum() >= 1
            # flagged tets are exactly the incident tets whose exact orientation changed
            Qn = np.array([[q10(base[v, a], off[v, 3 * side + a]) for a in range(3)] for v in range(len(base))])
            Q0 = np.array([[q10(base[v, a], 0.0) for a in range(3)] for v in range(len(base))])
            for tt in range(len(tets)):
                d_new = frac_det([[int(Qn[tets[tt][k + 1]][a] - Qn[tets[tt][0]][a]) for k in range(3)] for a in range(3)])
                d_old = frac_det([[int(Q0[tets[tt][k + 1]][a] - Q0[tets[tt][0]][a]) for k in range(3)] for a in range(3)])
                changed = (d_new > 0) != (d_old > 0) or d_new == 0
                assert flags[side, tt] == changed
                if changed:
                    assert tt in inc
            # severity = sum |signed volume| (mm^3) of the violating tets (App. A.4)
            exp = 0.0
            for tt in np.nonzero(flags[side])[0]:
                d_new = frac_det([[int(Qn[tets[tt][k + 1]][a] - Qn[tets[tt][0]][a]) for k in range(3)] for a in range(3)])
                exp += abs(float(d_new)) / 6 / 1024 ** 3 * 1.5 ** 3
            assert sev == pytest.approx(exp, rel=1e-12)


def test_small_moves_inside_link_do_not_fold():
    dims = (12, 12, 12)
    g = [-0.5, 3.5, 7.5, 11.5]
    base, tets = kuhn_lattice_mesh(g, g, g)
    I = blob_volume(dims, 1)
    orc = make_oracle(dims, I, I, base.astype(np.float32), tets)
    off = np.zeros((len(base), 6), np.float32)
    off[21] = [0.3, -0.2, 0.1, -0.4, 0.2, 0.3]
    assert orc.check_folds(off)[0] == 0


def test_zero_volume_counts_as_fold():
    """zero signed volume is a violation."""
    dims = (8, 8, 8)
    base = np.array([[-0.5, -0.5, -0.5], [7.5, -0.5, -0.5], [-0.5, 7.5, -0.5], [-0.5, -0.5, 7.5]], np.float32)
    tets = np.array([[0, 1, 2, 3]], np.int32)
    I = blob_volume(dims, 1)
    orc = make_oracle(dims, I, I, base, tets)
    off = np.zeros((4, 6), np.float32)
    off[3, 2] = -8.0  # vertex 3 into the z = -0.5 plane on the source side
    cnt, sev, flags = orc.check_folds(off)
    assert cnt == 1 and flags[0, 0] == 1 and sev == 0.0


def test_degenerate_base_rejected():
    dims = (8, 8, 8)
    base = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], np.float32)
    with pytest.raises(ValueError):
        make_oracle(dims, blob_volume(dims, 1), blob_volume(dims, 1), base, np.array([[0, 1, 2, 3]], np.int32))


def test_empty_sample_set_flag():
    """A mesh entirely outside the image has no samples: objectives NaN + F_EMPTY (O11)."""
    dims = (8, 8, 8)
    base = np.array([[20, 20, 20], [24, 20, 20], [20, 24, 20], [20, 20, 24]], np.float32)
    I = blob_volume(dims, 1)
    orc = make_oracle(dims, I, I, base, np.array([[0, 1, 2, 3]], np.int32))
    obj, acc = orc.eval(np.zeros((4, 6), np.float32))
    assert acc.n_samples == 0 and acc.flags & O.F_EMPTY and np.isnan(obj).all()


def test_domain_flag():
    dims = (8, 8, 8)
    base, tets = random_tiny_mesh(dims, 4, 1)
    I = blob_volume(dims, 1)
    orc = make_oracle(dims, I, I, base, tets)
    off = np.zeros((len(base), 6), np.float32)
    off[9, 4] = 900.0
    obj, acc = orc.eval(off)
    assert acc.flags & O.F_DOMAIN and np.isnan(obj).all()


# --------------------------------------------------------------------------- partial (O10)
def test_partial_equals_full_and_move_back(wl):
    """Partial delta on the dependent tets == full re-evaluation (1e-12); move-and-back."""
    for idx in (1, 2):
        w = wl(idx)
        orc = O.Oracle.from_workload(w)
        rng = np.random.default_rng(idx)
        for k in (1, 3, 7):
            base_obj, base_acc = orc.eval(w.offsets[k])
            for ns in (1, 2, 5):
                S = rng.choice(w.N, size=ns, replace=False).astype(np.int32)
                nv = w.offsets[k][S] + rng.normal(0, 0.4, size=(ns, 6)).astype(np.float32)
                fixed6 = np.concatenate([w.fixed_axes, w.fixed_axes], 1)[S]
                nv = np.where(fixed6, w.offsets[k][S], nv).astype(np.float32)
                obj, acc = orc.eval_partial(w.offsets[k], base_acc, S, nv)
                full_off = w.offsets[k].copy()
                full_off[S] = nv
                fobj, facc = orc.eval(full_off)
                assert acc.n_samples == facc.n_samples and acc.folds == facc.folds
                # the coverage check (a9) is defined for full evaluations only
                assert acc.flags == facc.flags & ~O.F_COVERAGE
                for a, b in ((acc.h_sum, facc.h_sum), (acc.g_sum, facc.g_sum),
                             (acc.m_sum, facc.m_sum), (acc.severity, facc.severity)):
                    assert a == pytest.approx(b, rel=1e-12, abs=1e-9)
                # move back
                bobj, bacc = orc.eval_partial(full_off, acc, S, w.offsets[k][S])
                assert bacc.n_samples == base_acc.n_samples
                assert bacc.h_sum == pytest.approx(base_acc.h_sum, rel=1e-12)
                assert bacc.g_sum == pytest.approx(base_acc.g_sum, rel=1e-12)


def test_coverage_flag_detects_gaps_and_overlaps():
    """Row a9 coverage check: per-side owned-sample counts vs the base mesh's.

    Moving a hull vertex inward leaves lattice points of the image uncovered
    (gap); folding an interior vertex covers some points twice (overlap).
    Identity and tangential hull motion keep the counts.
    """
    dims = (12, 12, 12)
    g = [-0.5, 3.5, 7.5, 11.5]
    base, tets = kuhn_lattice_mesh(g, g, g)
    base = base.astype(np.float32)
    I = blob_volume(dims, 3)
    orc = make_oracle(dims, I, I, base, tets)
    off = np.zeros((len(base), 6), np.float32)
    assert orc.eval(off)[1].flags == 0
    # corner (0,0,0) moved inward on the target side: the hull shrinks -> gap
    gap = off.copy()
    gap[0, 3:] = [2.0, 2.0, 2.0]
    _, acc = orc.eval(gap)
    assert acc.flags & O.F_COVERAGE and acc.n_samples < 2 * 12 ** 3
    # fold of an interior vertex on the source side: overlap (and a fold)
    j = 1 * 16 + 1 * 4 + 1
    t = int(np.nonzero((tets == j).any(1))[0][0])
    others = [v for v in tets[t] if v != j]
    c = base[others].astype(np.float64).mean(0)
    fold = off.copy()
    fold[j, :3] = (2 * c - base[j]) - base[j]
    _, acc = orc.eval(fold)
    assert acc.folds > 0 and acc.flags & O.F_COVERAGE


def test_sample_map_accessor_sums_to_h_sum(wl):
    """The test accessor orc_sample_map (per-voxel h, fg) re-states orc_eval's samples: on C2
    the per-voxel h of both sides sum to acc.h_sum, every voxel is sampled once per side
    (unfolded, hull at the image extent), and h follows the case rules of L318-322."""
    w = wl(2)
    orc = O.Oracle.from_workload(w)
    k = 5
    _, acc = orc.eval(w.offsets[k])
    tot = 0.0
    for side in (0, 1):
        h, fg = orc.sample_map(w.offsets[k], side)
        assert (fg != 255).all() and not np.isnan(h).any()
        tot += h.sum()
        a = (w.I_s if side == 0 else w.I_t).ravel()
        # the case rules of L318-322: both background -> 0, exactly one background -> 1
        assert (h[(a == 0) & (fg == 0)] == 0.0).all()
        assert (h[(a == 0) != (fg == 0)] == 1.0).all()
        assert ((a == 0) != (fg == 0)).sum() > 0
    assert tot == pytest.approx(acc.h_sum, rel=1e-12)

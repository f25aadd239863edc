"""Pins of the oracle's Sobol-in-tetrahedron sampler (NEXT-1, App. A.2
L744-751; readings S1..S9 in DESIGN.md §3) against things other than itself:
scipy's Sobol generator, published FNV-1a / SplitMix64 test vectors, math.log,
the Dirichlet(1,1,1,1) moments of the -log normalisation, exact tet volumes
(Python integers), closed-form objectives, and the partial == full invariant.
"""
import math

import numpy as np
import pytest
from scipy.stats import qmc

from oracle import oracle as O
from synth import kuhn_lattice_mesh
from tests.helpers import make_oracle, q10
from tests.test_oracle_pins import _translation_problem


# --------------------------------------------------------------------------- S1-S5 generator
def test_sobol_points_equal_scipy_unscrambled():
    """S1/S2: the first 4096 points equal scipy.stats.qmc.Sobol(d=4, scramble=False)."""
    n = 4096
    ours = O.sobol_points(n).astype(np.uint64)
    ref = qmc.Sobol(d=4, scramble=False).random(n) * 2.0 ** 32
    assert np.array_equal(ours, ref.astype(np.uint64))


def test_fnv1a_and_splitmix_published_vectors():
    """S3/S4: FNV-1a 64 and SplitMix64 against their published test vectors."""
    assert O.fnv1a64(b"") == 0xCBF29CE484222325
    assert O.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert O.fnv1a64(b"foobar") == 0x85944171F73967E8
    assert O.splitmix64(0) == 0xE220A8397B1DCDAF  # first output of SplitMix64 seeded with 0


def test_tet_seed_is_fnv_of_le_int32_coordinates():
    """S3: seed = FNV-1a over the 12 little-endian int32 Q.10 coordinates; masks from SplitMix64."""
    Q = np.array([[0, 0, 0], [1024, 0, 0], [0, 2048, 5], [-7, 3, 4096]], dtype=np.int64)
    seed, masks = O.tet_seed(Q)
    assert seed == O.fnv1a64(Q.astype("<i4").tobytes())
    for j in range(4):
        assert masks[j] == O.splitmix64((seed + j) % 2 ** 64) >> 32
    Q2 = Q.copy()
    Q2[3, 2] += 1
    assert O.tet_seed(Q2)[0] != seed


def test_neg_log_vs_math_log():
    """S5: the fixed-operation -log agrees with libm's log to 2 ulp over (0, 1)."""
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.integers(0, 2 ** 32, size=20000, dtype=np.uint64),
                         np.array([0, 1, 2, 2 ** 31 - 1, 2 ** 31, 2 ** 32 - 2, 2 ** 32 - 1], np.uint64)])
    for x in xs:
        u = (int(x) + 0.5) * 2.0 ** -32
        ref = -math.log(u)
        got = O.neg_log(int(x))
        assert abs(got - ref) <= 2 * math.ulp(ref)


# --------------------------------------------------------------------------- S6-S7 points in a tet
def _one_tet_problem(Qv, n=16):
    dims = (n, n, n)
    I = np.full((n, n, n), 0.5, np.float32)
    base = (np.asarray(Qv, dtype=np.float64) / 1024.0).astype(np.float32)
    tets = np.array([[0, 1, 2, 3]], np.int32)
    orc = make_oracle(dims, I, I, base, tets)
    return orc, np.zeros((4, 6), np.float32)


def test_barycentrics_on_simplex_and_dirichlet_moments():
    """S7: lambda >= 0, sum 1 (1e-12); over many points E[l_j] = 1/4, E[l_j^2] = 1/10
    (uniform on the simplex = Dirichlet(1,1,1,1), the paper's 'uniform spread')."""
    Qv = [[1024, 1024, 1024], [13 * 1024, 1024, 1024], [1024, 13 * 1024, 1024], [1024, 1024, 13 * 1024]]
    orc, off = _one_tet_problem(Qv)
    orc.set_sampler(1, 1.0)
    lams = []
    for k in range(4096):
        d = orc.sobol_debug(off, 0, 0, k)
        lam = d["lam"]
        assert (lam >= 0).all() and abs(lam.sum() - 1.0) < 1e-12
        # the point is the barycentric combination of the vertices
        X = np.asarray(Qv, float) / 1024.0
        assert np.allclose(d["p"], lam @ X, rtol=0, atol=1e-12)
        lams.append(lam)
    lams = np.array(lams)
    assert np.allclose(lams.mean(0), 0.25, atol=2e-3)
    assert np.allclose((lams ** 2).mean(0), 0.1, atol=2e-3)
    # second moments of the point cloud = those of the uniform tet (closed form)
    X = np.asarray(Qv, float) / 1024.0
    pts = lams @ X
    c = X.mean(0)
    cov_ref = (np.einsum("ki,kj->ij", X - c, X - c)) / 20.0  # uniform tet covariance
    assert np.allclose(np.cov(pts.T, bias=True), cov_ref, atol=0.02 * np.abs(cov_ref).max())


def test_sample_count_is_rounded_volume():
    """S6: N = floor(rate |Delta| / (6 1024^3) + 1/2), |Delta| exact (Python integers)."""
    rng = np.random.default_rng(3)
    for trial in range(20):
        Qv = rng.integers(0, 15 * 1024, size=(4, 3))
        M = [[int(Qv[k][a] - Qv[0][a]) for a in range(3)] for k in (1, 2, 3)]
        det = (M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1])
               - M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0])
               + M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]))
        if det == 0:
            continue
        if det < 0:
            Qv[[1, 2]] = Qv[[2, 1]]
        orc, off = _one_tet_problem(Qv)
        for rate in (1.0, 0.37, 2.5):
            orc.set_sampler(1, rate)
            N = orc.sobol_debug(off, 0, 0, 0)["N"]
            exact = abs(det) * rate / (6 * 1024 ** 3)
            assert abs(N - exact) <= 0.5 + 1e-9
    # doubling the volume doubles N (+-1)
    Qv = np.array([[0, 0, 0], [10240, 0, 0], [0, 10240, 0], [0, 0, 10240]])
    orc1, off = _one_tet_problem(Qv + 1024)
    Qv2 = Qv.copy()
    Qv2[3, 2] *= 2
    orc2, _ = _one_tet_problem(Qv2 + 1024)
    orc1.set_sampler(1)
    orc2.set_sampler(1)
    n1 = orc1.sobol_debug(off, 0, 0, 0)["N"]
    n2 = orc2.sobol_debug(off, 0, 0, 0)["N"]
    assert abs(n2 - 2 * n1) <= 1


def test_same_coordinates_same_samples():
    """App. A.2: identical tet coordinates give identical sample points."""
    Qv = np.array([[2048, 2048, 2048], [9000, 2100, 2000], [2500, 9500, 2600], [3000, 2900, 10000]])
    orc_a, off = _one_tet_problem(Qv)
    orc_b, _ = _one_tet_problem(Qv)
    orc_a.set_sampler(1)
    orc_b.set_sampler(1)
    for k in (0, 1, 17, 500):
        da, db = orc_a.sobol_debug(off, 0, 0, k), orc_b.sobol_debug(off, 0, 0, k)
        assert np.array_equal(da["p"], db["p"])
    # moving one vertex re-seeds the tet: the first point's barycentrics change
    off2 = off.copy()
    off2[2, 0] = 1.0 / 1024.0
    assert not np.array_equal(orc_a.sobol_debug(off2, 0, 0, 0)["lam"], orc_a.sobol_debug(off, 0, 0, 0)["lam"])


# --------------------------------------------------------------------------- S8-S9 objectives
def _lattice_problem(n=16, lo=2.0, hi=13.0, cells=3):
    g = np.linspace(lo, hi, cells + 1)
    base, tets = kuhn_lattice_mesh(g, g, g)
    return (n, n, n), base.astype(np.float32), tets


def test_identity_with_equal_volumes_gives_zero_intensity_term():
    """I_s = I_t and the identity map: a = b at every sample, so f_int = 0 exactly."""
    dims, base, tets = _lattice_problem()
    rng = np.random.default_rng(5)
    I = rng.uniform(0.0, 1.0, size=(16, 16, 16)).astype(np.float32)
    I[I < 0.3] = 0.0
    orc = make_oracle(dims, I, I, base, tets)
    orc.set_sampler(1, 1.0)
    off = np.zeros((len(base), 6), np.float32)
    off[:, :3] = np.round(rng.normal(0, 0.3, size=(len(base), 3)) * 1024) / 1024
    off[:, 3:] = off[:, :3]
    obj, acc = orc.eval(off)
    assert acc.n_samples > 0 and obj[1] == 0.0


def test_linear_volume_translation_closed_form():
    """I(x) = c.x + d > 0 everywhere, target mesh = source mesh + t: trilinear is exact on
    linear functions, so a - b = -c.t (source side) / +c.t (target side) at every sample and
    f_int = (c.t)^2 (S8/S9: both values interpolated at the mapped points)."""
    dims, base, tets = _lattice_problem()
    n = 16
    c = np.array([0.011, 0.017, 0.023])
    z, y, x = np.meshgrid(range(n), range(n), range(n), indexing="ij")
    I = (c[0] * x + c[1] * y + c[2] * z + 0.05).astype(np.float32)
    t = np.array([1.0, -0.5, 0.75])
    off = np.zeros((len(base), 6), np.float32)
    off[:, 3:] = t
    orc = make_oracle(dims, I, I, base, tets)
    orc.set_sampler(1, 1.0)
    obj, acc = orc.eval(off)
    # fp32 voxel values: I is c.x + d only to fp32 rounding (relative 6e-8 of <= 1)
    assert obj[1] == pytest.approx(float(c @ t) ** 2, rel=2e-5)
    assert acc.n_samples > 1000


def test_integer_translation_gives_zero_objectives_sobol():
    """The exact-zero translation phantom of O4 in Sobol mode: f_mag = 0 exactly, f_int and
    f_guid zero to rounding (T p = p + t up to one rounding of the barycentric sum)."""
    dims, I_s, I_t, cs, ct, base, tets, off = _translation_problem()
    orc = make_oracle(dims, I_s, I_t, base, tets, cs=cs, ct=ct, r_mm=3.0)
    orc.set_sampler(1, 1.0)
    obj, acc = orc.eval(off)
    assert acc.n_samples > 0
    assert obj[0] == 0.0
    assert abs(obj[1]) < 1e-20 and abs(obj[2]) < 1e-18
    off2 = off.copy()
    off2[:, 3:] = off2[:, :3]
    assert orc.eval(off2)[0][2] > 0.0  # not vacuous


def test_sample_total_is_sum_of_rounded_volumes(wl):
    """n_samples = sum over tets and sides of the rounded volumes (exact integer volumes)."""
    w = wl(1)
    orc = O.Oracle.from_workload(w)
    orc.set_sampler(1, 0.5)
    k = 3
    _, acc = orc.eval(w.offsets[k])
    total = 0
    for t in range(w.T):
        for s in range(2):
            Q = [[q10(w.base[j][a], w.offsets[k][j, 3 * s + a]) for a in range(3)] for j in w.tets[t]]
            M = [[Q[i][a] - Q[0][a] for a in range(3)] for i in (1, 2, 3)]
            det = (M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1])
                   - M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0])
                   + M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]))
            total += math.floor(float(abs(det)) * (0.5 / 6442450944.0) + 0.5)
    assert acc.n_samples == total


def test_sobol_partial_equals_full(wl):
    """O10 in Sobol mode: the dependent-tet delta equals full re-evaluation (1e-12)."""
    w = wl(1)
    orc = O.Oracle.from_workload(w)
    orc.set_sampler(1, 1.0)
    rng = np.random.default_rng(11)
    for k in (1, 2):
        _, base_acc = orc.eval(w.offsets[k])
        S = rng.choice(w.N, size=3, replace=False).astype(np.int32)
        fixed6 = np.concatenate([w.fixed_axes, w.fixed_axes], 1)[S]
        nv = np.where(fixed6, w.offsets[k][S],
                      w.offsets[k][S] + rng.normal(0, 0.3, size=(3, 6))).astype(np.float32)
        obj, acc = orc.eval_partial(w.offsets[k], base_acc, S, nv)
        full = w.offsets[k].copy()
        full[S] = nv
        fobj, facc = orc.eval(full)
        assert acc.n_samples == facc.n_samples
        for a, b in ((acc.h_sum, facc.h_sum), (acc.g_sum, facc.g_sum), (acc.m_sum, facc.m_sum)):
            assert a == pytest.approx(b, rel=1e-12, abs=1e-12)
        # no coverage flag in Sobol mode (a9 is defined on the voxel-centre sample set)
        assert not (facc.flags & O.F_COVERAGE)


def test_magnitude_independent_of_sampler(wl):
    w = wl(1)
    orc = O.Oracle.from_workload(w)
    a = orc.eval(w.offsets[2])[0][0]
    orc.set_sampler(1, 1.0)
    assert orc.eval(w.offsets[2])[0][0] == a

"""Pins of the oracle's fold repair (NEXT-2, §4.3.1; readings
P1..P7 in DESIGN.md §3) against things other than itself: scipy's normal
distribution and libm's log for the generator, the point-to-plane distance in
numpy for sigma, the Fig. 2 fold construction, exact signed volumes (Python
integers) and the invariants the paper states ("the change with the best
constraint improvement is selected, if present").
"""
import math

import numpy as np
import pytest
from scipy import stats

from oracle import oracle as O
from synth import kuhn_lattice_mesh
from tests.helpers import blob_volume, frac_det, make_oracle, q10


# --------------------------------------------------------------------------- P5 generator
def test_det_ln_vs_math_log():
    rng = np.random.default_rng(1)
    for r in np.concatenate([rng.uniform(1e-12, 1.0, 5000), [1.0, 0.5, 1e-300, 0.999999999]]):
        ref = math.log(r)
        assert abs(O.det_ln(r) - ref) <= 2 * math.ulp(ref) + 1e-300


def test_gaussian_generator_is_standard_normal():
    """Marsaglia polar draws: KS test against N(0, 1), moments.  (Streams are
    splitmix64(key + counter): keys are themselves SplitMix64 outputs (P5).)"""
    g = np.concatenate([O.gauss(O.splitmix64(k), 4000) for k in range(5)])
    assert stats.kstest(g, "norm").pvalue > 1e-3
    assert abs(g.mean()) < 0.03 and abs(g.var() - 1.0) < 0.04
    assert abs(stats.kurtosis(g)) < 0.15
    # deterministic per key, different across keys
    assert np.array_equal(O.gauss(7, 10), O.gauss(7, 10))
    assert not np.array_equal(O.gauss(7, 10), O.gauss(8, 10))


# --------------------------------------------------------------------------- problems
def _lattice(n=12):
    g = [-0.5, 3.5, 7.5, 11.5]
    base, tets = kuhn_lattice_mesh(g, g, g)
    base = base.astype(np.float32)
    dims = (n, n, n)
    I = blob_volume(dims, 1)
    return dims, base, tets, make_oracle(dims, I, I, base, tets)


def _hull_fixed(base):
    """P8: hull points keep the axes normal to their boundary planes."""
    return (base <= -0.5) | (base >= 11.5)


def _fig2_offsets(base, tets, j, t, side, depth=1.0):
    """Fig. 2 (L347-373): push point j through the opposite face of tet t (depth 1 = its
    mirror image through the opposite face's centroid)."""
    others = [v for v in tets[t] if v != j]
    c = base[others].astype(np.float64).mean(0)
    off = np.zeros((len(base), 6), np.float32)
    off[j, 3 * side:3 * side + 3] = depth * 2 * (c - base[j])
    return off


def _exact_side_severity(base, tets, off, side, ref):
    Q = np.array([[q10(base[v, a], off[v, 3 * side + a]) for a in range(3)] for v in range(len(base))])
    folds, sev = 0, 0.0
    for t in range(len(tets)):
        d = frac_det([[int(Q[tets[t][k + 1]][a] - Q[tets[t][0]][a]) for k in range(3)] for a in range(3)])
        if (d > 0) - (d < 0) != ref[t]:
            folds += 1
            sev += abs(float(d)) / 6 / 1024 ** 3 * 1.5 ** 3
    return folds, sev


# --------------------------------------------------------------------------- P4 sigma
def test_sigma_is_half_min_distance_to_opposite_planes():
    dims, base, tets, orc = _lattice()
    j = 21  # interior lattice point (1, 1, 1)
    off = np.zeros((len(base), 6), np.float32)
    inc = np.nonzero((tets == j).any(1))[0]
    P = base.astype(np.float64)
    dmin = np.inf
    for t in inc:
        o = [v for v in tets[t] if v != j]
        n = np.cross(P[o[1]] - P[o[0]], P[o[2]] - P[o[0]])
        dmin = min(dmin, abs(np.dot(P[j] - P[o[0]], n)) / np.linalg.norm(n))
    assert orc.repair_sigma(off, 0, j) == pytest.approx(0.5 * dmin, rel=1e-12)


# --------------------------------------------------------------------------- P1-P7 behaviour
def test_fold_free_input_is_unchanged():
    dims, base, tets, orc = _lattice()
    rng = np.random.default_rng(2)
    off = (rng.normal(0, 0.2, size=(len(base), 6)) * (np.abs(base) < 11)[:, [0, 1, 2, 0, 1, 2]]).astype(np.float32)
    assert orc.check_folds(off)[0] == 0
    new, moved, aborted = orc.repair(off, 123, 0)
    assert moved == 0 and aborted == 0 and np.array_equal(new, off)


@pytest.mark.parametrize("side", [0, 1])
@pytest.mark.parametrize("depth", [0.6, 1.0])
def test_fig2_fold_is_improved_never_worsened(side, depth):
    dims, base, tets, orc = _lattice()
    ref = np.array([orc.ref_sign(t) for t in range(len(tets))])
    j = 21
    inc = np.nonzero((tets == j).any(1))[0]
    fixed = _hull_fixed(base)
    n_fixed = 0
    for t in inc[:6]:
        off = _fig2_offsets(base, tets, j, t, side, depth)
        f0, s0 = _exact_side_severity(base, tets, off, side, ref)
        assert f0 >= 1
        for seed in (1, 2, 3):
            new, moved, aborted = orc.repair(off, seed, 5, fixed)
            f1, s1 = _exact_side_severity(base, tets, new, side, ref)
            # strictly better (lexicographic: folds, then severity), other side untouched,
            # fixed axes untouched
            assert (f1, s1) < (f0, s0)
            assert np.array_equal(new[:, 3 * side:3 * side + 3][fixed], off[:, 3 * side:3 * side + 3][fixed])
            assert np.array_equal(new[:, 3 * (1 - side):3 * (1 - side) + 3], off[:, 3 * (1 - side):3 * (1 - side) + 3])
            # only vertices of folded tets move
            movers = np.nonzero((new != off).any(1))[0]
            folded_vertices = set()
            for tt in range(len(tets)):
                Q = [[q10(base[v, a], off[v, 3 * side + a]) for a in range(3)] for v in tets[tt]]
                d = frac_det([[Q[k + 1][a] - Q[0][a] for k in range(3)] for a in range(3)])
                if (d > 0) - (d < 0) != ref[tt]:
                    folded_vertices |= set(int(v) for v in tets[tt])
            assert set(movers.tolist()) <= folded_vertices
            assert moved == len(movers)
            n_fixed += f1 == 0


def test_repair_deterministic_and_seeded(wl):
    w = wl(1)
    orc = O.Oracle.from_workload(w)
    k = 7  # a forced-fold solution
    assert orc.check_folds(w.offsets[k])[0] > 0
    a = orc.repair(w.offsets[k], 99, k)
    b = orc.repair(w.offsets[k], 99, k)
    c = orc.repair(w.offsets[k], 100, k)
    assert np.array_equal(a[0], b[0]) and a[1:] == b[1:]
    assert not np.array_equal(a[0], c[0])


def test_repair_reduces_folds_on_workload(wl):
    """Over the forced-fold solutions of C1/C2 the summed (folds, severity) never rises."""
    for idx in (1, 2):
        w = wl(idx)
        orc = O.Oracle.from_workload(w)
        for k in range(7, w.P, 16):
            c0, s0, _ = orc.check_folds(w.offsets[k])
            fixed = w.fixed_axes
            new, moved, aborted = orc.repair(w.offsets[k], 2024, k, fixed)
            c1, s1, _ = orc.check_folds(new)
            assert (c1, s1) <= (c0, s0 + 1e-12)
            assert moved + aborted >= 1
            fx6 = np.concatenate([fixed, fixed], 1)
            assert np.array_equal(new[fx6], w.offsets[k][fx6])

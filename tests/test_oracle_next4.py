"""Pins of the oracle's rasterizer reuse (NEXT-4): per-tet object fractions and
the elasticity factor c_delta (App. A.1), and the deformation
vector field export (§5.4).  Readings E1..E3 in DESIGN.md §3.  Pinned to
the owner map (itself pinned to a Fraction brute force), a numpy label rule,
the paper's worked example ("a fraction of 0.4 for the object", L731) and
closed-form displacement fields.
"""
import numpy as np
import pytest

from oracle import oracle as O
from synth import random_tiny_mesh
from tests.helpers import blob_volume, make_oracle
from tests.test_oracle_pins import _affine_problem


def _labels_np(masks, M):
    """E1 in numpy: 1 + lowest set bit below M, 0 for none."""
    lab = np.zeros(masks.shape, np.int64)
    for b in reversed(range(M)):
        lab = np.where((masks >> b) & 1, b + 1, lab)
    return lab


def _masks(dims, seed):
    rng = np.random.default_rng(seed)
    n = dims[0]
    z, y, x = np.meshgrid(*(np.arange(d) for d in dims[::-1]), indexing="ij")
    m = np.zeros(dims[::-1], np.uint8)
    m |= ((x - n / 3) ** 2 + (y - n / 2) ** 2 + (z - n / 2) ** 2 < (n / 4) ** 2).astype(np.uint8)
    m |= ((x > 2 * n / 3) & (y < n / 2)).astype(np.uint8) << 1
    m |= (rng.uniform(size=m.shape) < 0.2).astype(np.uint8) << 2  # overlaps the others
    return m


def test_label_counts_match_owner_map():
    dims = (10, 10, 10)
    base, tets = random_tiny_mesh(dims, 10, 4)
    I = blob_volume(dims, 2)
    orc = make_oracle(dims, I, I, base, tets)
    masks = _masks(dims, 1)
    rng = np.random.default_rng(3)
    off = np.zeros((len(base), 6), np.float32)
    off[8:] = np.round(rng.normal(0, 0.3, size=(len(base) - 8, 6)) * 1024) / 1024
    lab = _labels_np(masks.reshape(-1), 3)
    for side in (0, 1):
        own = orc.owner_map(off, side)
        exp = np.zeros((len(tets), 4), np.int64)
        ok = own >= 0
        np.add.at(exp, (own[ok], lab[ok]), 1)
        got = orc.label_counts(off, side, masks, 3)
        assert np.array_equal(got, exp)
        # the base mesh covers the image exactly once: column sums = label histogram
    got0 = orc.label_counts(None, 0, masks, 3)
    assert np.array_equal(got0.sum(0), np.bincount(lab, minlength=4))


def test_elasticity_worked_example_and_trivial_cases():
    """App. A.1: "a fraction of 0.4 for the object" -> c = 0.4 f + 0.6 * 1.0."""
    dims = (10, 10, 10)
    base = np.array([[-0.5, -0.5, -0.5], [9.5, -0.5, -0.5], [-0.5, 9.5, -0.5], [-0.5, -0.5, 9.5]], np.float32)
    tets = np.array([[0, 1, 2, 3]], np.int32)
    I = blob_volume(dims, 2)
    orc = make_oracle(dims, I, I, base, tets)
    none = np.zeros((10, 10, 10), np.uint8)
    assert orc.elasticity(none, [10.0])[0] == 1.0  # no object -> 1.0
    own = orc.owner_map(np.zeros((4, 6), np.float32), 0)
    idx = np.nonzero(own == 0)[0]
    full = none.reshape(-1).copy()
    full[idx] = 1
    assert orc.elasticity(full, [10.0])[0] == pytest.approx(10.0, rel=1e-7)  # fully inside
    # exactly 40 % of the tet's voxels in the object
    k = int(round(0.4 * len(idx)))
    part = none.reshape(-1).copy()
    part[idx[:k]] = 1
    frac = k / len(idx)
    assert orc.elasticity(part, [10.0])[0] == pytest.approx(frac * 10.0 + (1 - frac) * 1.0, rel=1e-7)
    # priority: a voxel in objects 0 and 1 counts for object 0 only
    both = part | (1 << 1)
    c = orc.elasticity(both, [10.0, 0.5])[0]
    assert c == pytest.approx(frac * 10.0 + (1 - frac) * 0.5, rel=1e-7)


def test_dvf_identity_translation_affine():
    """E3: T(q) - q in mm; identity -> 0, translation -> t * spacing, global affine ->
    (A q + b - q) * spacing (forward) and (A^-1 (q - b) - q) * spacing (inverse)."""
    dims, base, tets, off, A, b = _affine_problem()
    I = blob_volume(dims, 5)
    sp = np.array([1.5, 1.25, 2.0])
    orc = make_oracle(dims, I, I, base, tets, spacing=sp)
    n = dims[0]
    z, y, x = np.meshgrid(range(n), range(n), range(n), indexing="ij")
    q = np.stack([x.ravel(), y.ravel(), z.ravel()], 1).astype(np.float64)
    d, cov = orc.dvf(np.zeros_like(off), 0)
    assert cov.all() and not d.any()
    t = np.array([0.5, -1.25, 2.0], np.float32)
    off_t = np.zeros_like(off)
    off_t[:, 3:] = t
    d, cov = orc.dvf(off_t, 0)
    assert cov.all()
    assert np.array_equal(d, np.broadcast_to((t * sp).astype(np.float32), d.shape))
    d, cov = orc.dvf(off, 0)
    assert cov.all()
    np.testing.assert_allclose(d, (q @ A.T + b - q) * sp, rtol=0, atol=1e-6)
    d1, cov1 = orc.dvf(off, 1)
    inside = cov1.astype(bool)
    assert inside.sum() > 0.8 * n ** 3
    qi = q[inside]
    np.testing.assert_allclose(d1[inside], ((qi - b) @ np.linalg.inv(A).T - qi) * sp, rtol=0, atol=1e-6)

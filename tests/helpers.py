"""Test-side helpers: small hand-built problems and exact (Fraction) references.

The exact references here use a different algorithm from the oracle's (a
Fraction Gaussian-elimination solve for barycentric coordinates instead of
integer face normals) so that a mistake in one does not hide in the other.
"""
from fractions import Fraction

import numpy as np


def frac_solve(A, b):
    """Solve A x = b exactly (A: 3x3 Fractions, b: 3 Fractions) by Gauss-Jordan."""
    M = [[Fraction(A[i][j]) for j in range(3)] + [Fraction(b[i])] for i in range(3)]
    for c in range(3):
        p = next(r for r in range(c, 3) if M[r][c] != 0)
        M[c], M[p] = M[p], M[c]
        piv = M[c][c]
        M[c] = [v / piv for v in M[c]]
        for r in range(3):
            if r != c and M[r][c] != 0:
                f = M[r][c]
                M[r] = [vr - f * vc for vr, vc in zip(M[r], M[c])]
    return [M[i][3] for i in range(3)]


def frac_inverse(A):
    cols = [frac_solve(A, [1 if i == j else 0 for i in range(3)]) for j in range(3)]
    return [[cols[j][i] for j in range(3)] for i in range(3)]  # inv[i][j]


def frac_det(A):
    """Exact determinant by fraction-free elimination (not cofactor expansion)."""
    M = [[Fraction(v) for v in row] for row in A]
    det = Fraction(1)
    for c in range(3):
        p = next((r for r in range(c, 3) if M[r][c] != 0), None)
        if p is None:
            return Fraction(0)
        if p != c:
            M[c], M[p] = M[p], M[c]
            det = -det
        det *= M[c][c]
        for r in range(c + 1, 3):
            f = M[r][c] / M[c][c]
            M[r] = [vr - f * vc for vr, vc in zip(M[r], M[c])]
    return det


def q10(base, off):
    """Canonical fixed point per DESIGN.md reading O1, recomputed in Python."""
    v = 1024.0 * float(np.float32(base)) + 1024.0 * float(np.float32(off))
    return int(round(v))  # Python round() = round-half-even


class FracTet:
    """Exact barycentric machinery for one tet given its 4 vertices in Q units."""

    def __init__(self, Qv):
        self.Qv = [[int(c) for c in v] for v in Qv]
        v0 = self.Qv[0]
        E = [[self.Qv[k + 1][a] - v0[a] for k in range(3)] for a in range(3)]  # columns = edges
        self.det = frac_det(E)
        self.inv = frac_inverse(E) if self.det != 0 else None

    def bary(self, p):
        """lambda_0..3 of point p (Fractions, Q units) and their gradients (rows)."""
        v0 = self.Qv[0]
        d = [Fraction(p[a]) - v0[a] for a in range(3)]
        lam123 = [sum(self.inv[i][a] * d[a] for a in range(3)) for i in range(3)]
        grads = [[self.inv[i][a] for a in range(3)] for i in range(3)]
        g0 = [-(grads[0][a] + grads[1][a] + grads[2][a]) for a in range(3)]
        return [1 - sum(lam123)] + lam123, [g0] + grads

    def owns(self, q):
        """Ownership of lattice point q (voxel units) under q + (e, e^2, e^3) (reading O3)."""
        if self.det == 0:
            return False
        lam, grads = self.bary([1024 * c for c in q])
        for lk, gk in zip(lam, grads):
            if lk > 0:
                continue
            if lk < 0:
                return False
            g = next((v for v in gk if v != 0), 0)
            if not g > 0:
                return False
        return True


def axis_set_frac(x, n):
    """Contributing lattice indices of the clamped trilinear footprint (reading O5/O6)."""
    if x <= 0:
        return [0]
    if x >= n - 1:
        return [n - 1]
    fl = x.numerator // x.denominator
    if fl == x:
        return [int(fl)]
    return [int(fl), int(fl) + 1]


def make_oracle(dims, I_s, I_t, base, tets, cs=None, ct=None, r_mm=None, spacing=(1.5, 1.5, 1.5),
                c_delta=None, spoke_mode=0):
    from oracle.oracle import Oracle
    cs = list(cs) if cs else []
    ct = list(ct) if ct else []

    def csr(cc):
        off = np.concatenate([[0], np.cumsum([len(c) for c in cc])]).astype(np.int64)
        xyz = (np.vstack(cc).astype(np.float32) if cc and off[-1] > 0
               else np.zeros((1, 3), np.float32))
        return off, xyz

    cs_off, cs_xyz = csr(cs)
    ct_off, ct_xyz = csr(ct)
    if r_mm is None:
        r_mm = 0.025 * dims[0] * spacing[0]
    return Oracle(dims, np.asarray(spacing, float), I_s, I_t, cs_off, cs_xyz, ct_off, ct_xyz,
                  r_mm, base, tets, c_delta, spoke_mode)


def blob_volume(dims, seed, frac_zero=0.4, margin=0):
    """Random non-negative volume with exact zeros (background) and positive values."""
    rng = np.random.default_rng(seed)
    nx, ny, nz = dims
    v = rng.uniform(0.05, 1.0, size=(nz, ny, nx)).astype(np.float32)
    v[rng.uniform(size=v.shape) < frac_zero] = 0.0
    if margin:
        m = np.zeros_like(v, dtype=bool)
        m[margin:nz - margin, margin:ny - margin, margin:nx - margin] = True
        v[~m] = 0.0
    return v

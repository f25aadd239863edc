"""Empty-space skipping counted exactly (run with -m gpu).

k_raster counts, without sweeping them, the rows of an item whose voxels are all
quiet: background (I = 0) on the sampled side, no band entry (every D_i >= r), and
the other volume zero within Chebyshev distance R - 1, R = ceil(max|U| / 1024) + 2
for the item (U = the per-vertex displacement in Q.10).  The test rebuilds that
classification independently of the kernel -- row intervals from the oracle's owner
map, band bits from the oracle's distance maps, zero radii from scipy's chessboard
distance transform, Q.10 vertices from the oracle's canonicalisation -- and compares
the number of quiet-row samples with the kernel's profiling counter (`skipped`),
exactly.  The objectives of the same call are checked against the oracle, so the
samples counted this way are known to contribute h = 0 and no guidance term.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)

from scipy import ndimage  # noqa: E402

from oracle.oracle import Oracle, canon  # noqa: E402
from paper_2303_04873_b200 import morea  # noqa: E402
from tests.test_gpu_parity import _assert_acc, _assert_obj, _ctx  # noqa: E402

RMIN, RMAX, ZR_CAP = 2, 15, 15


def _quiet_samples(w, orc, k):
    nx, ny, nz = w.dims
    vols = [np.asarray(w.I_s, np.float32).reshape(nz, ny, nx), np.asarray(w.I_t, np.float32).reshape(nz, ny, nx)]
    K = len(w.pairs)
    # per-tet radius from the Q.10 vertices of both sides
    N = w.base.shape[0]
    Q = np.zeros((2, N, 3), np.int64)
    for s in range(2):
        for j in range(N):
            for a in range(3):
                Q[s, j, a] = canon(w.base[j][a], w.offsets[k][j][3 * s + a])
    U = np.abs(Q[1] - Q[0])                       # (N, 3)
    maxU = U[np.asarray(w.tets)].max(axis=(1, 2))  # per tet
    R = (maxU + 1023) // 1024 + 2
    total = 0
    for s in range(2):
        other = vols[1 - s]
        if (other != 0).any():
            zr = ndimage.distance_transform_cdt(other == 0, metric="chessboard")
        else:
            zr = np.full(other.shape, ZR_CAP)
        zr = np.minimum(zr, ZR_CAP)
        band = np.zeros((nz, ny, nx), bool)
        for i in range(K):
            band |= orc.distance_map(s, i).reshape(nz, ny, nx) < orc.r
        q = np.where((vols[s] != 0) | band, 0, zr)
        first, last = {}, {}
        for r in range(RMIN, RMAX + 1):
            nq = q < r
            anyq = nq.any(axis=2)
            first[r] = np.where(anyq, nq.argmax(axis=2), nx)
            last[r] = np.where(anyq, nx - 1 - nq[:, :, ::-1].argmax(axis=2), -1)
        om = orc.owner_map(w.offsets[k], s).reshape(nz, ny, nx)
        z, y, x = np.nonzero(om >= 0)
        t = om[z, y, x].astype(np.int64)
        key = (t * nz + z) * ny + y
        u, inv, cnt = np.unique(key, return_inverse=True, return_counts=True)
        xmin = np.full(len(u), nx)
        xmax = np.full(len(u), -1)
        np.minimum.at(xmin, inv, x)
        np.maximum.at(xmax, inv, x)
        assert np.array_equal(xmax - xmin + 1, cnt)  # a tet's row is one interval
        tt, zz, yy = u // (nz * ny), (u // ny) % nz, u % ny
        Rt = R[tt]
        quiet = np.zeros(len(u), bool)
        for r in range(RMIN, RMAX + 1):
            m = Rt == r
            f, l = first[r][zz[m], yy[m]], last[r][zz[m], yy[m]]
            quiet[m] = (xmax[m] < f) | (xmin[m] > l)
        total += int(cnt[quiet].sum())
    return total


@pytest.mark.parametrize("idx,ks", [(1, [0, 3]), (2, [0, 5, 63])])
def test_quiet_row_samples_counted_exactly(wl, idx, ks):
    w = wl(idx)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    ctx.prof_enable(True)
    seen = 0
    for k in ks:
        if orc.check_folds(w.offsets[k])[0] > 0:
            continue  # owner maps of folded solutions overlap; rows are not single intervals
        seen += 1
        obj = np.empty((1, 3), np.float64)
        acc = np.empty(1, morea.ACC_DTYPE)
        ctx.prof_read()
        ctx.eval_full(np.ascontiguousarray(w.offsets[k:k + 1]), obj, acc, None)
        st = ctx.prof_read()
        want = _quiet_samples(w, orc, k)
        assert want > 0, (w.name, k)
        assert st["skipped"] == want, (w.name, k, st["skipped"], want)
        o_obj, o_acc = orc.eval(w.offsets[k])
        _assert_acc(acc[0], o_acc, f"{w.name} sol {k}")
        _assert_obj(obj[0], o_obj, f"{w.name} sol {k}")
    assert seen >= 1
    ctx.close()

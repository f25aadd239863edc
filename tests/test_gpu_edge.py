"""GPU edge cases (run with -m gpu): long rows that overflow one row-start
bitmap window (more than 2048 samples per 32-row chunk), the minimum volume,
sizes at the gather-texture limits of the layout, background-only volumes, and
empty requests.  Same bar as tests/test_gpu_parity.py."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)

from synth import kuhn_lattice_mesh, random_tiny_mesh  # noqa: E402
from tests.helpers import blob_volume, make_oracle  # noqa: E402
from tests.test_gpu_parity import DEV, _assert_acc, _assert_obj, _ctx_raw, _gpu_full  # noqa: E402


def _check(dims, I_s, I_t, base, tets, offs, cs=None, ct=None):
    ctx = _ctx_raw(dims, I_s, I_t, base, tets, cs, ct)
    orc = make_oracle(dims, I_s, I_t, base, tets, cs=cs, ct=ct)
    obj, acc, _, _, _ = _gpu_full(ctx, offs)
    for k in range(offs.shape[0]):
        o_obj, o_acc = orc.eval(offs[k])
        _assert_acc(acc[k], o_acc, f"sol {k}")
        _assert_obj(obj[k], o_obj, f"sol {k}")
    for side in (0, 1):
        own = np.empty(ctx.V, np.int32)
        ctx.owner_map(offs[-1], side, own)
        assert np.array_equal(own, orc.owner_map(offs[-1], side))
    return ctx


def _offsets(base, P, seed, scale, fixed=None):
    rng = np.random.default_rng(seed)
    offs = np.round(rng.normal(0, scale, size=(P, len(base), 6)) * 1024) / 1024
    if fixed is not None:
        offs[:, fixed] = 0.0
    offs[0] = 0.0
    return offs.astype(np.float32)


def test_long_rows_span_several_bitmap_windows():
    """dims 700 x 6 x 5 with tets spanning hundreds of voxels in x: a 32-row chunk
    holds > 2048 samples (up to ~22 000), so the row-start bitmap is swept in several windows."""
    dims = (700, 6, 5)
    g = [np.linspace(-0.5, d - 0.5, 3) for d in dims]
    base, tets = kuhn_lattice_mesh(*g)
    base = base.astype(np.float32)
    hull = (np.abs(base + 0.5) < 1e-6) | (np.abs(base - (np.array(dims) - 0.5)) < 1e-6)
    I_s = blob_volume(dims, 11)
    I_t = blob_volume(dims, 12)
    offs = _offsets(base, 4, 3, 0.4)
    offs[:, :, :3][:, hull] = 0.0
    offs[:, :, 3:][:, hull] = 0.0
    _check(dims, I_s, I_t, base, tets, offs)


def test_minimum_volume():
    dims = (2, 2, 2)
    base = np.array([[x, y, z] for z in (-0.5, 1.5) for y in (-0.5, 1.5) for x in (-0.5, 1.5)], np.float32)
    from scipy.spatial import Delaunay
    tets = Delaunay(base.astype(np.float64)).simplices.astype(np.int32)
    I = np.array([0.0, 0.5, 0.25, 0.0, 1.0, 0.0, 0.75, 0.125], np.float32).reshape(2, 2, 2)
    offs = np.zeros((2, 8, 6), np.float32)
    offs[1, :, 3:] = 0.25
    _check(dims, I, I[::-1].copy(), base, tets, offs)


def test_background_only_and_guidance_pairs():
    dims = (20, 18, 16)
    base, tets = random_tiny_mesh(dims, 12, 5)
    I0 = np.zeros(dims[::-1], np.float32)
    rng = np.random.default_rng(4)
    cs = [rng.uniform(3, 14, size=(30, 3)).astype(np.float32) for _ in range(3)]
    ct = [(c + rng.normal(0, 0.5, size=c.shape)).astype(np.float32) for c in cs]
    offs = _offsets(base, 3, 6, 0.2)
    offs[:, :8] = 0.0
    _check(dims, I0, I0, base, tets, offs, cs, ct)


def test_empty_requests_are_noops(wl):
    w = wl(1)
    ctx = _ctx_raw(w.dims, w.I_s, w.I_t, w.base, w.tets)
    obj = torch.full((1, 3), 7.0, dtype=torch.float64, device=DEV)
    acc = torch.zeros((1, 6), dtype=torch.int64, device=DEV)
    off = torch.zeros((0, w.N, 6), dtype=torch.float32, device=DEV)
    ctx.eval_full(off, obj, acc, None)
    ctx.eval_partial(off, acc, np.array([0], np.int32), np.zeros(0, np.int32), torch.zeros(0, device=DEV),
                     None, obj, acc)
    torch.cuda.synchronize()
    assert float(obj[0, 0]) == 7.0


def test_border_band_positions_nonzero_border():
    """Positions in (-1, 0) and (n-1, n) on every axis read the one-voxel replicated
    border of the gather textures without the explicit clamp (O5 through the
    padding); positions beyond it take the clamping instantiation.  Volumes and
    distance maps are non-zero at the border, so a wrong border texel shows."""
    dims = (20, 18, 16)
    base, tets = random_tiny_mesh(dims, 14, 8)
    I_s = blob_volume(dims, 21, frac_zero=0.2)
    I_t = blob_volume(dims, 22, frac_zero=0.2)
    rng = np.random.default_rng(9)
    cs = [rng.uniform(0, 15, size=(40, 3)).astype(np.float32) for _ in range(2)]
    ct = [(c + rng.normal(0, 0.7, size=c.shape)).astype(np.float32) for c in cs]
    N = len(base)
    offs = np.zeros((6, N, 6), np.float32)
    offs[1] = _offsets(base, 2, 10, 0.25)[1]
    offs[1, :8] = 0.0                       # interior moves, hull at the image extent
    offs[2, :, 3:] = [0.4375, -0.6875, 0.9375]   # translation inside the border band
    offs[3, :, :3] = [-0.875, 0.8125, -0.5]      # same on the source side
    offs[4, :, 3:] = [2.25, -1.5, 3.0]           # beyond the band: clamp instantiation
    offs[5] = offs[1]
    offs[5, :, 3:] += np.array([0.3125, -0.25, 0.1875], np.float32)  # generic map into the band
    _check(dims, I_s, I_t, base, tets, offs, cs, ct)


def test_plain_load_path_parity(wl, monkeypatch):
    """Volumes beyond the 2D gather-texture limits (e.g. 512 x 512 x 128: (ny+2)(nz+2)
    rows > 32768) run k_raster / k_sobol with plain loads and the explicit O5 clamp.
    MOREA_NO_TEX forces that path on C2: full and partial evaluation, owner maps and
    the Sobol sampler against the oracle."""
    from oracle.oracle import Oracle
    from paper_2303_04873_b200 import morea
    from synth import fos_plan, partial_request
    w = wl(2)
    monkeypatch.setenv("MOREA_NO_TEX", "1")
    ctx = morea.Context.from_workload(w, device=0)
    orc = Oracle.from_workload(w)
    obj, acc, tc, off, acc_d = _gpu_full(ctx, w.offsets, cache=True)
    sols = (0, 1, 7, 23, w.P - 1)
    for k in sols:
        o_obj, o_acc = orc.eval(w.offsets[k])
        _assert_acc(acc[k], o_acc, f"plain C2 sol {k}")
        _assert_obj(obj[k], o_obj, f"plain C2 sol {k}")
    for side in (0, 1):
        own = np.empty(ctx.V, np.int32)
        ctx.owner_map(w.offsets[1], side, own)
        assert np.array_equal(own, orc.owner_map(w.offsets[1], side))
    plan = fos_plan(w.tets, w.N)
    go, ch, nv = partial_request(w, plan, "edges4", 0)
    G = len(go) - 1
    pobj = torch.empty((w.P * G, 3), dtype=torch.float64, device=DEV)
    pacc = torch.empty((w.P * G, 6), dtype=torch.int64, device=DEV)
    ctx.eval_partial(off, acc_d, go, ch, torch.from_numpy(nv).to(DEV), torch.from_numpy(tc).to(DEV), pobj, pacc)
    torch.cuda.synchronize()
    p_obj, p_acc = pobj.cpu().numpy(), morea.acc_to_numpy(pacc)
    for k in (1, 7):
        base_o = orc.eval(w.offsets[k])[1]
        for g in (0, G - 1):
            S = ch[go[g]:go[g + 1]]
            o_obj, o_acc = orc.eval_partial(w.offsets[k], base_o, S, nv[k, go[g]:go[g + 1]])
            _assert_acc(p_acc[k * G + g], o_acc, f"plain partial sol {k} group {g}")
            _assert_obj(p_obj[k * G + g], o_obj, f"plain partial sol {k} group {g}")
    ctx.set_sampler(morea.SAMPLER_SOBOL, 1.0)
    orc.set_sampler(morea.SAMPLER_SOBOL, 1.0)
    obj, acc, _, _, _ = _gpu_full(ctx, w.offsets[:8])
    for k in (0, 1, 5):
        o_obj, o_acc = orc.eval(w.offsets[k])
        _assert_acc(acc[k], o_acc, f"plain Sobol sol {k}")
        _assert_obj(obj[k], o_obj, f"plain Sobol sol {k}")

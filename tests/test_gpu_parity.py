"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle (run with -m gpu).

Bar (BASELINE.json north_star): bit-exact voxel ownership and fold flags;
objectives within 1e-5 relative (fp32 values, fp64 accumulation); integer
outputs (sample counts, fold counts, flags) exact.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.oracle import Oracle  # noqa: E402
from paper_2303_04873_b200 import morea  # noqa: E402
from synth import fos_plan, kuhn_lattice_mesh, partial_request, random_tiny_mesh  # noqa: E402
from tests.helpers import blob_volume, make_oracle  # noqa: E402

DEV = torch.device("cuda:0")
RTOL = 1e-5


def _ctx(w):
    return morea.Context.from_workload(w, device=0)


def _ctx_raw(dims, I_s, I_t, base, tets, cs=None, ct=None, r_mm=None, spacing=(1.5, 1.5, 1.5),
             c_delta=None, spoke_mode=0):
    cs = list(cs) if cs else []
    ct = list(ct) if ct else []

    def csr(cc):
        off = np.concatenate([[0], np.cumsum([len(c) for c in cc])]).astype(np.int64)
        xyz = np.vstack(cc).astype(np.float32) if cc and off[-1] > 0 else np.zeros((1, 3), np.float32)
        return off, xyz

    cso, csx = csr(cs)
    cto, ctx_ = csr(ct)
    if r_mm is None:
        r_mm = 0.025 * dims[0] * spacing[0]
    c = morea.Context(0)
    c.load_images(dims, spacing, I_s, I_t, cso, csx, cto, ctx_, r_mm)
    c.set_mesh(base, tets, c_delta, spoke_mode)
    return c


def _gpu_full(ctx, offsets, cache=False):
    P = offsets.shape[0]
    off = torch.from_numpy(np.ascontiguousarray(offsets, np.float32)).to(DEV)
    obj = torch.empty((P, 3), dtype=torch.float64, device=DEV)
    acc = torch.empty((P, 6), dtype=torch.int64, device=DEV)
    tc = torch.empty((P, ctx.T, 4), dtype=torch.float64, device=DEV) if cache else None
    ctx.eval_full(off, obj, acc, tc)
    torch.cuda.synchronize()
    return obj.cpu().numpy(), morea.acc_to_numpy(acc), (tc.cpu().numpy() if cache else None), off, acc


def _assert_obj(g_obj, o_obj, what=""):
    for i in range(3):
        if np.isnan(o_obj[i]):
            assert np.isnan(g_obj[i]), what
        else:
            assert g_obj[i] == pytest.approx(o_obj[i], rel=RTOL, abs=1e-12), (what, i, g_obj, o_obj)


def _assert_acc(g, o, what=""):
    assert g["n_samples"] == o.n_samples, what
    assert g["folds"] == o.folds, what
    assert g["flags"] == o.flags, what
    for k in ("h_sum", "g_sum", "m_sum", "severity"):
        assert g[k] == pytest.approx(getattr(o, k), rel=RTOL, abs=1e-9), (what, k)


# ---------------------------------------------------------------------------- a0: maps
@pytest.mark.parametrize("idx", [1, 2])
def test_distance_maps_bitexact(wl, idx):
    w = wl(idx)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    for s in (0, 1):
        for i in range(len(w.pairs)):
            np.testing.assert_array_equal(ctx.distance_map(s, i), orc.distance_map(s, i))


def test_distance_maps_anisotropic_bitexact():
    dims = (13, 11, 9)
    sp = (1.5, 0.8, 2.25)
    rng = np.random.default_rng(8)
    cs = [rng.uniform(-1, 12, size=(57, 3)).astype(np.float32), rng.uniform(0, 8, size=(3, 3)).astype(np.float32)]
    ct = [rng.uniform(0, 10, size=(20, 3)).astype(np.float32), np.array([[4.0, 5.0, 6.0]], np.float32)]
    I = blob_volume(dims, 1)
    base, tets = random_tiny_mesh(dims, 5, 3)
    ctx = _ctx_raw(dims, I, I, base, tets, cs, ct, spacing=sp)
    orc = make_oracle(dims, I, I, base, tets, cs=cs, ct=ct, spacing=sp)
    for s in (0, 1):
        for i in range(2):
            np.testing.assert_array_equal(ctx.distance_map(s, i), orc.distance_map(s, i))


# ---------------------------------------------------------------------------- a4: ownership
@pytest.mark.parametrize("idx", [1, 2])
def test_owner_map_bitexact_workloads(wl, idx):
    w = wl(idx)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    for k in sorted(set([0, 1, 7, w.P - 1])):
        for side in (0, 1):
            np.testing.assert_array_equal(ctx.owner_map(w.offsets[k], side), orc.owner_map(w.offsets[k], side),
                                          err_msg=f"{w.name} sol {k} side {side}")


def test_owner_map_bitexact_tie_heavy_integer_kuhn():
    """Integer-vertex Kuhn mesh: faces, edges, vertices and hull faces hit voxel centres."""
    dims = (10, 10, 10)
    base, tets = kuhn_lattice_mesh([0, 4, 8], [0, 4, 8], [0, 4, 8])
    base = base.astype(np.float32)
    I = blob_volume(dims, 7)
    ctx = _ctx_raw(dims, I, I, base, tets)
    orc = make_oracle(dims, I, I, base, tets)
    rng = np.random.default_rng(0)
    for trial in range(4):
        off = np.zeros((len(base), 6), np.float32)
        if trial:
            # integer moves of interior points keep ties on lattice planes
            off[13] = rng.integers(-1, 2, size=6)
        for side in (0, 1):
            np.testing.assert_array_equal(ctx.owner_map(off, side), orc.owner_map(off, side))


@pytest.mark.parametrize("seed", range(6))
def test_owner_map_bitexact_random_meshes(seed):
    dims = (14, 12, 10)
    base, tets = random_tiny_mesh(dims, 25, seed)
    rng = np.random.default_rng(seed)
    off = np.zeros((len(base), 6), np.float32)
    off[8:] = rng.normal(0, 0.4, size=(len(base) - 8, 6))  # folds allowed
    I = blob_volume(dims, seed)
    ctx = _ctx_raw(dims, I, I, base, tets)
    orc = make_oracle(dims, I, I, base, tets)
    for side in (0, 1):
        np.testing.assert_array_equal(ctx.owner_map(off, side), orc.owner_map(off, side))


# ---------------------------------------------------------------------------- a2/a9: folds
@pytest.mark.parametrize("idx", [1, 2, 3, 4])
def test_fold_flags_bitexact(wl, idx):
    w = wl(idx)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    P = w.P
    cnt = np.zeros(P, np.int32)
    sev = np.zeros(P, np.float64)
    flags = np.zeros((P, 2, w.T), np.uint8)
    ctx.check_folds(w.offsets, cnt, sev, flags)
    for k in range(P):
        oc, os_, of = orc.check_folds(w.offsets[k])
        assert cnt[k] == oc
        np.testing.assert_array_equal(flags[k], of)
        assert sev[k] == pytest.approx(os_, rel=1e-12, abs=1e-12)


# ---------------------------------------------------------------------------- full evaluation
@pytest.mark.parametrize("idx", [1, 2])
def test_eval_full_parity_all_solutions(wl, idx):
    w = wl(idx)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    g_obj, g_acc, tc, _, _ = _gpu_full(ctx, w.offsets, cache=True)
    for k in range(w.P):
        o_obj, o_acc = orc.eval(w.offsets[k])
        _assert_acc(g_acc[k], o_acc, f"{w.name} sol {k}")
        _assert_obj(g_obj[k], o_obj, f"{w.name} sol {k}")
    # per-tet contributions of a few solutions
    for k in (0, 1, w.P - 1):
        rec = orc.eval_tets(w.offsets[k])
        np.testing.assert_array_equal(tc[k, :, 2], rec[:, 2] + rec[:, 3])
        np.testing.assert_allclose(tc[k, :, 0], rec[:, 0], rtol=RTOL, atol=1e-9)
        np.testing.assert_allclose(tc[k, :, 1], rec[:, 1], rtol=RTOL, atol=1e-9)
        np.testing.assert_allclose(tc[k, :, 3], rec[:, 4], rtol=1e-9, atol=1e-12)


@pytest.mark.slow
def test_eval_full_parity_c3_subset(wl):
    w = wl(3)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    g_obj, g_acc, _, _, _ = _gpu_full(ctx, w.offsets)
    for k in (0, 1, 7, 100, 255):
        o_obj, o_acc = orc.eval(w.offsets[k])
        _assert_acc(g_acc[k], o_acc, f"C3 sol {k}")
        _assert_obj(g_obj[k], o_obj, f"C3 sol {k}")


@pytest.mark.slow
def test_eval_full_parity_c4_full_size_sampled(wl):
    """Paper scale (C4, P = 512) in the launch configuration bench.py times: the whole
    population is evaluated in one call; sampled solutions are checked in full and
    sampled tets of every 64th solution one by one against the oracle."""
    w = wl(4)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    g_obj, g_acc, tc, _, _ = _gpu_full(ctx, w.offsets, cache=True)
    for k in (1, 300):
        o_obj, o_acc = orc.eval(w.offsets[k])
        _assert_acc(g_acc[k], o_acc, f"C4 sol {k}")
        _assert_obj(g_obj[k], o_obj, f"C4 sol {k}")
    rng = np.random.default_rng(0)
    for k in range(0, w.P, 64):
        sub = rng.choice(w.T, 12, replace=False).astype(np.int32)
        rec = orc.eval_tets(w.offsets[k], sub)
        np.testing.assert_array_equal(tc[k, sub, 2], rec[:, 2] + rec[:, 3])
        np.testing.assert_allclose(tc[k, sub, 0], rec[:, 0], rtol=RTOL, atol=1e-9)
        np.testing.assert_allclose(tc[k, sub, 1], rec[:, 1], rtol=RTOL, atol=1e-9)
    # properties at any size: unfolded solutions own every voxel exactly once per side
    cnt = np.zeros(w.P, np.int32)
    ctx.check_folds(w.offsets, cnt, None, None)
    unf = cnt == 0
    assert (g_acc["n_samples"][unf] == 2 * w.V).all()
    assert np.isfinite(g_obj[unf]).all()


# ---------------------------------------------------------------------------- edge cases
def test_exact_landing_positions_take_the_slow_path():
    """x = 2 q + b lands on lattice points for every sample (all positions ambiguous
    for the fp32 filter): the exact fallback must reproduce the oracle."""
    from tests.test_oracle_pins import _affine_problem
    dims, base, tets, off, A, b = _affine_problem(12, A=2.0 * np.eye(3), b=np.array([-6.0, -5.0, -4.0]))
    I_s = blob_volume(dims, 13, frac_zero=0.5)
    I_t = blob_volume(dims, 14, frac_zero=0.5)
    ctx = _ctx_raw(dims, I_s, I_t, base, tets)
    orc = make_oracle(dims, I_s, I_t, base, tets)
    g_obj, g_acc, _, _, _ = _gpu_full(ctx, off[None])
    o_obj, o_acc = orc.eval(off)
    _assert_acc(g_acc[0], o_acc)
    _assert_obj(g_obj[0], o_obj)
    # generic affine (never integer) too
    dims, base, tets, off, A, b = _affine_problem()
    ctx = _ctx_raw(dims, I_s, I_t, base, tets)
    orc = make_oracle(dims, I_s, I_t, base, tets)
    g_obj, g_acc, _, _, _ = _gpu_full(ctx, off[None])
    o_obj, o_acc = orc.eval(off)
    _assert_acc(g_acc[0], o_acc)
    _assert_obj(g_obj[0], o_obj)


def test_integer_translation_exact_zeros():
    from tests.test_oracle_pins import _translation_problem
    dims, I_s, I_t, cs, ct, base, tets, off = _translation_problem()
    ctx = _ctx_raw(dims, I_s, I_t, base, tets, cs, ct, r_mm=3.0)
    g_obj, g_acc, _, _, _ = _gpu_full(ctx, off[None])
    assert (g_obj[0] == 0.0).all()
    assert g_acc["n_samples"][0] > 0


def test_identity_is_voxelwise_h(wl):
    w = wl(2)
    ctx = _ctx(w)
    g_obj, _, _, _, _ = _gpu_full(ctx, w.offsets[:1])
    orc = Oracle.from_workload(w)
    o_obj, _ = orc.eval(w.offsets[0])
    assert g_obj[0][0] == 0.0
    assert g_obj[0][1] == pytest.approx(o_obj[1], rel=1e-7)  # exact positions; h in fp32, sum in fp64


def test_empty_and_domain_flags():
    dims = (8, 8, 8)
    I = blob_volume(dims, 1)
    base = np.array([[20, 20, 20], [24, 20, 20], [20, 24, 20], [20, 20, 24]], np.float32)
    tets = np.array([[0, 1, 2, 3]], np.int32)
    ctx = _ctx_raw(dims, I, I, base, tets)
    g_obj, g_acc, _, _, _ = _gpu_full(ctx, np.zeros((1, 4, 6), np.float32))
    assert g_acc["n_samples"][0] == 0 and g_acc["flags"][0] & morea.F_EMPTY and np.isnan(g_obj[0]).all()
    base, tets = random_tiny_mesh(dims, 4, 1)
    ctx = _ctx_raw(dims, I, I, base, tets)
    off = np.zeros((2, len(base), 6), np.float32)
    off[1, 9, 4] = 900.0
    g_obj, g_acc, _, _, _ = _gpu_full(ctx, off)
    assert g_acc["flags"][0] == 0 and g_acc["flags"][1] & morea.F_DOMAIN and np.isnan(g_obj[1]).all()


def test_api_errors():
    dims = (8, 8, 8)
    I = blob_volume(dims, 1)
    c = morea.Context(0)
    with pytest.raises(morea.MoreaError) as e:
        c.set_mesh(np.zeros((4, 3), np.float32), np.array([[0, 1, 2, 3]], np.int32))
    assert e.value.code == -2
    bad = I.copy()
    bad[0, 0, 0] = -1.0
    with pytest.raises(morea.MoreaError) as e:
        c.load_images(dims, (1, 1, 1), bad, I, [0], np.zeros((1, 3), np.float32), [0],
                      np.zeros((1, 3), np.float32))
    assert e.value.code == -1
    c.load_images(dims, (1, 1, 1), I, I, [0], np.zeros((1, 3), np.float32), [0], np.zeros((1, 3), np.float32))
    flat = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], np.float32)
    with pytest.raises(morea.MoreaError) as e:
        c.set_mesh(flat, np.array([[0, 1, 2, 3]], np.int32))
    assert e.value.code == -3
    # Sobol rate outside (0, 8]: per-tet point counts must stay 32-bit
    for bad_rate in (0.0, -1.0, 8.5, float("inf"), float("nan")):
        with pytest.raises(morea.MoreaError) as e:
            c.set_sampler(morea.SAMPLER_SOBOL, bad_rate)
        assert e.value.code == -1
    with pytest.raises(morea.MoreaError) as e:
        c.set_mesh(flat, np.array([[0, 1, 2, 9]], np.int32))
    assert e.value.code == -1


# ---------------------------------------------------------------------------- partial evaluation
@pytest.mark.parametrize("idx", [1, 2])
def test_eval_partial_parity(wl, idx):
    w = wl(idx)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    plan = fos_plan(w.tets, w.N)
    g_obj, g_acc, tc, off, acc = _gpu_full(ctx, w.offsets, cache=True)
    for kind in ("class", "edges4", "all"):
        go, ch, nv = partial_request(w, plan, kind, 1)
        G = len(go) - 1
        nvd = torch.from_numpy(nv).to(DEV)
        outs = []
        for cache in (None, torch.from_numpy(tc).to(DEV)):
            pobj = torch.empty((w.P * G, 3), dtype=torch.float64, device=DEV)
            pacc = torch.empty((w.P * G, 6), dtype=torch.int64, device=DEV)
            ctx.eval_partial(off, acc, go, ch, nvd, cache, pobj, pacc)
            torch.cuda.synchronize()
            outs.append((pobj.cpu().numpy(), morea.acc_to_numpy(pacc)))
        # cached == recomputed, bitwise
        np.testing.assert_array_equal(outs[0][0], outs[1][0])
        assert outs[0][1].tobytes() == outs[1][1].tobytes()
        p_obj, p_acc = outs[0]
        for k in sorted(set([0, 1, 7, w.P - 1])):
            base_o = orc.eval(w.offsets[k])[1]
            for g in range(G):
                S = ch[go[g]:go[g + 1]]
                o_obj, o_acc = orc.eval_partial(w.offsets[k], base_o, S, nv[k, go[g]:go[g + 1]])
                _assert_acc(p_acc[k * G + g], o_acc, f"{w.name} {kind} sol {k} group {g}")
                _assert_obj(p_obj[k * G + g], o_obj, f"{w.name} {kind} sol {k} group {g}")


def test_partial_equals_full_reevaluation(wl):
    """acc' from the delta == full GPU evaluation of the moved genotype (1e-12)."""
    w = wl(2)
    ctx = _ctx(w)
    plan = fos_plan(w.tets, w.N)
    _, _, tc, off, acc = _gpu_full(ctx, w.offsets, cache=True)
    go, ch, nv = partial_request(w, plan, "edges4", 0)
    G = len(go) - 1
    pobj = torch.empty((w.P * G, 3), dtype=torch.float64, device=DEV)
    pacc = torch.empty((w.P * G, 6), dtype=torch.int64, device=DEV)
    nvd = torch.from_numpy(nv).to(DEV)
    ctx.eval_partial(off, acc, go, ch, nvd, None, pobj, pacc)
    deps, dep_off = ctx.partial_deps()
    dep_out = torch.empty((w.P, len(deps), 4), dtype=torch.float64, device=DEV)
    ctx.eval_partial(off, acc, go, ch, nvd, torch.from_numpy(tc).to(DEV), pobj, pacc, dep_out)
    torch.cuda.synchronize()
    p_acc = morea.acc_to_numpy(pacc)
    for g in (0, G - 1):
        moved = w.offsets.copy()
        moved[:, ch[go[g]:go[g + 1]]] = nv[:, go[g]:go[g + 1]]
        f_obj, f_acc, f_tc, _, _ = _gpu_full(ctx, moved, cache=True)
        for k in range(w.P):
            a = p_acc[k * G + g]
            assert a["n_samples"] == f_acc["n_samples"][k] and a["folds"] == f_acc["folds"][k]
            for key in ("h_sum", "g_sum", "m_sum"):
                assert a[key] == pytest.approx(f_acc[key][k], rel=1e-12, abs=1e-9)
        # dep_cache_out holds the new per-tet contributions, bitwise equal to the full run's
        d = deps[dep_off[g]:dep_off[g + 1]]
        got = dep_out[:, dep_off[g]:dep_off[g + 1]].cpu().numpy()
        np.testing.assert_array_equal(got, f_tc[:, d])


# ---------------------------------------------------------------------------- determinism / sharding / host path
def test_determinism_sharding_and_host_pointers(wl):
    """Repeat runs bitwise equal; shards of the population (as ranks would evaluate
    them) bitwise equal to the whole batch; host-pointer inputs/outputs equal."""
    w = wl(2)
    ctx = _ctx(w)
    a = _gpu_full(ctx, w.offsets, cache=True)
    b = _gpu_full(ctx, w.offsets, cache=True)
    assert a[1].tobytes() == b[1].tobytes() and np.array_equal(a[2], b[2])
    for G in (2, 4, 8):
        parts = np.array_split(np.arange(w.P), G)
        accs = [_gpu_full(ctx, w.offsets[p])[1] for p in parts]
        assert np.concatenate(accs).tobytes() == a[1].tobytes()
    obj_h = np.empty((w.P, 3))
    acc_h = np.empty(w.P, morea.ACC_DTYPE)
    ctx.eval_full(np.ascontiguousarray(w.offsets), obj_h, acc_h, None)
    assert acc_h.tobytes() == a[1].tobytes()
    np.testing.assert_array_equal(obj_h, a[0])


def test_spoke_mode_and_cdelta(wl):
    w = wl(1)
    rng = np.random.default_rng(3)
    c = rng.uniform(0.5, 3.0, size=w.T).astype(np.float32)
    for mode in (0, 1):
        ctx = _ctx_raw(w.dims, w.I_s, w.I_t, w.base, w.tets, c_delta=c, spoke_mode=mode)
        orc = make_oracle(w.dims, w.I_s, w.I_t, w.base, w.tets, c_delta=c, spoke_mode=mode)
        g_obj, _, _, _, _ = _gpu_full(ctx, w.offsets)
        for k in range(w.P):
            assert g_obj[k][0] == pytest.approx(orc.eval(w.offsets[k])[0][0], rel=1e-10)


def test_coverage_flag_matches_oracle():
    """Row a9 coverage check on the GPU == oracle (gap from a moved hull vertex, overlap
    from a fold, none for identity / interior moves)."""
    dims = (12, 12, 12)
    g = [-0.5, 3.5, 7.5, 11.5]
    base, tets = kuhn_lattice_mesh(g, g, g)
    base = base.astype(np.float32)
    I = blob_volume(dims, 3)
    ctx = _ctx_raw(dims, I, I, base, tets)
    orc = make_oracle(dims, I, I, base, tets)
    offs = np.zeros((4, len(base), 6), np.float32)
    offs[1, 0, 3:] = [2.0, 2.0, 2.0]
    j = 1 * 16 + 1 * 4 + 1
    t = int(np.nonzero((tets == j).any(1))[0][0])
    others = [v for v in tets[t] if v != j]
    c = base[others].astype(np.float64).mean(0)
    offs[2, j, :3] = (2 * c - base[j]) - base[j]
    offs[3, j] = [0.3, -0.2, 0.1, -0.4, 0.2, 0.3]
    g_obj, g_acc, _, _, _ = _gpu_full(ctx, offs)
    for k in range(4):
        o_obj, o_acc = orc.eval(offs[k])
        _assert_acc(g_acc[k], o_acc, f"coverage case {k}")
    assert g_acc["flags"][0] == 0 and g_acc["flags"][3] == 0
    assert g_acc["flags"][1] & morea.F_COVERAGE and g_acc["flags"][2] & morea.F_COVERAGE

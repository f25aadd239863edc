"""GPU parity of the Sobol-in-tetrahedron sampler (NEXT-1, App. A.2
L744-751; readings S1..S9 in DESIGN.md §3) against the CPU oracle (run with -m gpu).

Bar: sample counts, fold counts and flags exact; objectives and per-tet sums
within 1e-5 relative.  Every decision on a sample position (clamp, corner set,
positivity of a and b) is taken on the oracle's exact fp64 position whenever
the fp32 fast path is within its error bound of a lattice plane; the
MOREA_SOBOL_FORCE_EXACT hook routes every sample through that fp64 path.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.oracle import Oracle  # noqa: E402
from paper_2303_04873_b200 import morea  # noqa: E402
from synth import fos_plan, partial_request  # noqa: E402
from tests.test_gpu_parity import DEV, RTOL, _assert_acc, _assert_obj, _ctx, _ctx_raw, _gpu_full  # noqa: E402
from tests.test_oracle_pins import _translation_problem  # noqa: E402


def _sobol_ctx(w, rate=1.0):
    c = _ctx(w)
    c.set_sampler(morea.SAMPLER_SOBOL, rate)
    return c


def _sobol_oracle(w, rate=1.0):
    o = Oracle.from_workload(w)
    o.set_sampler(1, rate)
    return o


@pytest.mark.parametrize("idx,sols", [(1, None), (2, (0, 1, 2, 5, 7, 23, 40, 63))])
def test_sobol_full_parity(wl, idx, sols):
    w = wl(idx)
    ctx = _sobol_ctx(w)
    orc = _sobol_oracle(w)
    obj, acc, _, _, _ = _gpu_full(ctx, w.offsets)
    for k in (range(w.P) if sols is None else sols):
        o_obj, o_acc = orc.eval(w.offsets[k])
        _assert_acc(acc[k], o_acc, f"C{idx} sol {k}")
        _assert_obj(obj[k], o_obj, f"C{idx} sol {k}")
        assert not (acc[k]["flags"] & 4)  # no coverage flag in Sobol mode


def test_sobol_per_tet_parity(wl):
    w = wl(2)
    ctx = _sobol_ctx(w)
    orc = _sobol_oracle(w)
    k = 3
    _, _, tc, _, _ = _gpu_full(ctx, w.offsets[k:k + 1], cache=True)
    rec = orc.eval_tets(w.offsets[k])
    n_o = rec[:, 2] + rec[:, 3]
    assert np.array_equal(tc[0, :, 2].astype(np.int64), n_o.astype(np.int64))
    # per-tet sums: 1e-5 relative, or an absolute slack of 1e-9 (h) / 1e-7 (g, mm^2) per sample
    for col, ocol, per in ((0, 0, 1e-9), (1, 1, 1e-7)):
        err = np.abs(tc[0, :, col] - rec[:, ocol])
        bound = RTOL * np.abs(rec[:, ocol]) + per * np.maximum(n_o, 1)
        assert (err <= bound).all(), (col, np.max(err / bound), np.argmax(err / bound))
    np.testing.assert_allclose(tc[0, :, 3], rec[:, 4], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("idx,sols", [(1, (0, 1, 3, 6)), (2, (1, 4))])
def test_sobol_exact_path_parity(wl, monkeypatch, idx, sols):
    """Every sample through the fp64 fallback: same decisions and sums as the oracle."""
    w = wl(idx)
    monkeypatch.setenv("MOREA_SOBOL_FORCE_EXACT", "1")
    ctx = _sobol_ctx(w)
    orc = _sobol_oracle(w)
    off = w.offsets[list(sols)]
    obj, acc, _, _, _ = _gpu_full(ctx, off)
    monkeypatch.delenv("MOREA_SOBOL_FORCE_EXACT")
    obj2, acc2, _, _, _ = _gpu_full(ctx, off)
    for j, k in enumerate(sols):
        o_obj, o_acc = orc.eval(w.offsets[k])
        _assert_acc(acc[j], o_acc, f"exact path C{idx} sol {k}")
        _assert_obj(obj[j], o_obj, f"exact path C{idx} sol {k}")
        # the fast path agrees with the exact path (decisions are the same by construction)
        assert acc2[j]["n_samples"] == acc[j]["n_samples"]
        assert acc2[j]["h_sum"] == pytest.approx(acc[j]["h_sum"], rel=1e-6)


@pytest.mark.parametrize("rate", [0.25, 3.0])
def test_sobol_rates(wl, rate):
    w = wl(1)
    ctx = _sobol_ctx(w, rate)
    orc = _sobol_oracle(w, rate)
    obj, acc, _, _, _ = _gpu_full(ctx, w.offsets)
    for k in range(w.P):
        o_obj, o_acc = orc.eval(w.offsets[k])
        _assert_acc(acc[k], o_acc, f"rate {rate} sol {k}")


def test_sobol_deterministic_and_mode_switch(wl):
    w = wl(2)
    ctx = _ctx(w)
    v_obj, v_acc, _, _, _ = _gpu_full(ctx, w.offsets[:8])
    ctx.set_sampler(morea.SAMPLER_SOBOL, 1.0)
    a_obj, a_acc, _, _, _ = _gpu_full(ctx, w.offsets[:8])
    b_obj, b_acc, _, _, _ = _gpu_full(ctx, w.offsets[:8])
    assert np.array_equal(a_obj, b_obj) and np.array_equal(a_acc, b_acc)
    assert not np.array_equal(a_obj[:, 1], v_obj[:, 1])  # a different sample set
    ctx.set_sampler(morea.SAMPLER_VOXEL)
    c_obj, c_acc, _, _, _ = _gpu_full(ctx, w.offsets[:8])
    assert np.array_equal(c_obj, v_obj) and np.array_equal(c_acc, v_acc)


def test_sobol_partial(wl):
    """Partial (colour class, cached and stateless) vs the oracle and vs full evaluation."""
    w = wl(2)
    ctx = _sobol_ctx(w)
    orc = _sobol_oracle(w)
    P = 16
    offs = np.ascontiguousarray(w.offsets[:P])
    obj, acc, tc, off_d, acc_d = _gpu_full(ctx, offs, cache=True)
    plan = fos_plan(w.tets, w.N)
    go, ch, nv = partial_request(w, plan, "class", 0)
    nv = np.ascontiguousarray(nv[:P])
    G = len(go) - 1
    nvd = torch.from_numpy(nv).to(DEV)
    tcd = torch.from_numpy(tc).to(DEV)
    res = []
    for cache in (tcd, None):
        pobj = torch.empty((P * G, 3), dtype=torch.float64, device=DEV)
        pacc = torch.empty((P * G, 6), dtype=torch.int64, device=DEV)
        ctx.eval_partial(off_d, acc_d, go, ch, nvd, cache, pobj, pacc)
        torch.cuda.synchronize()
        res.append((pobj.cpu().numpy(), morea.acc_to_numpy(pacc)))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    pobj, pacc = res[0]
    for k in (0, 3, 9):
        _, base = orc.eval(offs[k])
        for g in (0, G // 2, G - 1):
            o_obj, o_acc = orc.eval_partial(offs[k], base, ch[go[g]:go[g + 1]], nv[k, go[g]:go[g + 1]])
            _assert_acc(pacc[k * G + g], o_acc, f"partial sol {k} group {g}")
            _assert_obj(pobj[k * G + g], o_obj, f"partial sol {k} group {g}")


def test_sobol_integer_translation_zero():
    """The O4 translation phantom in Sobol mode: f_mag = 0, f_int and f_guid ~ 0."""
    dims, I_s, I_t, cs, ct, base, tets, off = _translation_problem()
    ctx = _ctx_raw(dims, I_s, I_t, base, tets, cs=cs, ct=ct, r_mm=3.0)
    ctx.set_sampler(morea.SAMPLER_SOBOL, 1.0)
    obj, acc, _, _, _ = _gpu_full(ctx, off[None])
    assert acc[0]["n_samples"] > 0
    assert obj[0][0] == 0.0
    assert abs(obj[0][1]) < 1e-12 and abs(obj[0][2]) < 1e-10


@pytest.mark.slow
def test_sobol_c3_sample(wl):
    w = wl(3)
    ctx = _sobol_ctx(w)
    orc = _sobol_oracle(w)
    sols = (1, 100)
    obj, acc, _, _, _ = _gpu_full(ctx, np.ascontiguousarray(w.offsets[list(sols)]))
    for j, k in enumerate(sols):
        o_obj, o_acc = orc.eval(w.offsets[k])
        _assert_acc(acc[j], o_acc, f"C3 sol {k}")
        _assert_obj(obj[j], o_obj, f"C3 sol {k}")

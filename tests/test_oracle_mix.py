"""Pins of the oracle's optimal mixing of one FOS colour class (NEXT-3, PAPER.md
§3; readings M1..M7 in DESIGN.md §3): the sampler against the
closed-form mean and covariance of mu + L z, and the acceptance rules replayed
independently with full evaluations (the mixing itself uses partial ones).
"""
import numpy as np
import pytest

from oracle import oracle as O
from synth import fos_plan


def model_from_population(offs, grp_off, changed, eps=1e-6):
    """Per-group mean and Cholesky factor of the population's group variables."""
    mus, Ls = [], []
    for g in range(len(grp_off) - 1):
        S = changed[grp_off[g]:grp_off[g + 1]]
        X = offs[:, S, :].reshape(offs.shape[0], -1).astype(np.float64)
        mu = X.mean(0)
        C = np.cov(X.T, bias=True) + eps * np.eye(X.shape[1])
        mus.append(mu)
        Ls.append(np.linalg.cholesky(C).ravel())
    return np.concatenate(mus), np.concatenate(Ls)


def test_mix_sampler_mean_and_covariance():
    """M1/M2: x = mu + L z with z ~ N(0, I): E x = mu, Cov x = L L^T."""
    rng = np.random.default_rng(0)
    d = 12
    mu = rng.normal(0, 1, d)
    Lc = np.tril(rng.normal(0, 0.3, (d, d)))
    Lc[np.diag_indices(d)] = np.abs(Lc[np.diag_indices(d)]) + 0.2
    xs = np.array([O.mix_sample(mu, Lc.ravel(), 5, 1, k, 3) for k in range(20000)])
    se = np.sqrt(np.diag(Lc @ Lc.T) / len(xs))
    assert np.all(np.abs(xs.mean(0) - mu) < 4 * se)
    np.testing.assert_allclose(np.cov(xs.T), Lc @ Lc.T, atol=0.05 * np.abs(Lc @ Lc.T).max())
    # deterministic per key
    assert np.array_equal(O.mix_sample(mu, Lc.ravel(), 5, 1, 7, 3), O.mix_sample(mu, Lc.ravel(), 5, 1, 7, 3))


def _class(w, ci=0):
    plan = fos_plan(w.tets, w.N)
    # plan: colour classes of FOS elements (edges); reuse the workload's request builder
    from synth import partial_request
    go, ch, _ = partial_request(w, plan, "class", ci)
    return np.asarray(go, np.int32), np.asarray(ch, np.int32)


def _replay(orc, w, off, acc, obj, go, ch, mu, Lc, fixed, archive, steer, seed, gen, k):
    """M1-M7 replayed with full evaluations."""
    state = off.copy()
    cur = np.array(obj, float)
    acc_flags = []
    mo = lo = 0
    for g in range(len(go) - 1):
        S = ch[go[g]:go[g + 1]]
        d = 6 * len(S)
        x = O.mix_sample(mu[mo:mo + d], Lc[lo:lo + d * d], seed, gen, k, g)
        mo += d
        lo += d * d
        cand = state.copy()
        for i in range(d):
            pt, c = S[i // 6], i % 6
            if not (fixed is not None and fixed[pt, c % 3]):
                cand[pt, c] = np.float32(x[i])
        cobj, cacc = orc.eval(cand)
        ok = cacc.folds == 0 and not (cacc.flags & (O.F_DOMAIN | O.F_EMPTY))
        if ok and steer > 0 and not cobj[2] <= steer:
            ok = False
        if ok:
            dom_parent = np.all(cobj <= cur) and np.any(cobj < cur)
            dominated = any(np.all(a <= cobj) and np.any(a < cobj) for a in archive)
            ok = dom_parent or not dominated
        acc_flags.append(int(ok))
        if ok:
            state, cur = cand, cobj
    return state, cur, np.array(acc_flags, np.uint8)


@pytest.mark.parametrize("steer", [0.0, 1e-30])
def test_mix_rules_replayed_with_full_evaluations(wl, steer):
    w = wl(1)
    orc = O.Oracle.from_workload(w)
    go, ch = _class(w)
    offs = w.offsets
    mu, Lc = model_from_population(offs, go, ch, eps=0.01)
    objs = np.array([orc.eval(offs[k])[0] for k in range(w.P)])
    archive = objs[[0, 2, 4]]
    n_acc = 0
    for k in (1, 2, 3, 5):
        obj, acc = orc.eval(offs[k])
        new, nacc, nobj, flags = orc.mix(offs[k], acc, obj, go, ch, mu, Lc, w.fixed_axes, archive, steer, 77, 3, k)
        r_state, r_obj, r_flags = _replay(orc, w, offs[k], acc, obj, go, ch, mu, Lc, w.fixed_axes, archive,
                                          steer, 77, 3, k)
        assert np.array_equal(flags, r_flags), k
        assert np.array_equal(new, r_state)
        np.testing.assert_allclose(nobj, r_obj, rtol=1e-9)
        # the carried accumulator equals a full evaluation of the final state
        fobj, facc = orc.eval(new)
        assert nacc.n_samples == facc.n_samples and nacc.folds == facc.folds
        assert nacc.h_sum == pytest.approx(facc.h_sum, rel=1e-9)
        assert nacc.g_sum == pytest.approx(facc.g_sum, rel=1e-9)
        assert nacc.m_sum == pytest.approx(facc.m_sum, rel=1e-9)
        fx6 = np.concatenate([w.fixed_axes, w.fixed_axes], 1)
        assert np.array_equal(new[fx6], offs[k][fx6])
        n_acc += flags.sum()
    if steer > 0:
        assert n_acc == 0
    else:
        assert n_acc > 0


def test_mix_identity_candidate_leaves_state(wl):
    """Zero-variance model at the parent: the offspring is the parent; state unchanged."""
    w = wl(1)
    orc = O.Oracle.from_workload(w)
    go, ch = _class(w)
    k = 2
    off = w.offsets[k]
    mu = np.concatenate([off[ch[go[g]:go[g + 1]]].astype(np.float64).ravel() for g in range(len(go) - 1)])
    Lc = np.concatenate([np.zeros(36 * (go[g + 1] - go[g]) ** 2) for g in range(len(go) - 1)])
    obj, acc = orc.eval(off)
    new, nacc, nobj, flags = orc.mix(off, acc, obj, go, ch, mu, Lc, None, np.zeros((0, 3)), 0.0, 1, 0, k)
    assert np.array_equal(new, off)
    assert nacc.h_sum == pytest.approx(acc.h_sum, rel=1e-12) and nacc.n_samples == acc.n_samples

"""GPU parity at the two paper-scale configurations (run with -m gpu).

- C5 (BASELINE.json configs[4]): P = 4096 solutions of the paper-scale volume,
  sharded the way bench.py shards them across ranks (contiguous blocks of
  P/G, `shard_bounds`).  On one GPU each shard is evaluated by its own call;
  the shard outputs must be bitwise equal to one unsharded call (SURVEY.md
  §8(e) correctness invariant), fold flags bit-exact for every solution, and
  sampled solutions of every shard within 1e-5 of the oracle.
- C4 (configs[3]): the partial-evaluation sweep over FOS sizes (SURVEY.md
  §8(d): 1 edge, 4 and 16 edges of one colour class, one whole colour class,
  all 600 points), cached and stateless, against the oracle on sampled
  solutions and groups.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.oracle import Oracle  # noqa: E402
from paper_2303_04873_b200 import morea  # noqa: E402
from paper_2303_04873_b200.distributed import shard_bounds  # noqa: E402
from synth import fos_plan, partial_request  # noqa: E402
from tests.test_gpu_parity import DEV, _assert_acc, _assert_obj, _ctx, _gpu_full  # noqa: E402


def test_c5_sharded_parity(wl):
    w = wl(5)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    # one unsharded call over all 4096 solutions
    g_obj, g_acc, _, _, _ = _gpu_full(ctx, w.offsets)
    G = 8
    checked = []
    for r in range(G):
        s0, s1 = shard_bounds(w.P, G, r)
        s_obj, s_acc, _, _, _ = _gpu_full(ctx, w.offsets[s0:s1])
        # shard == unsharded, bitwise
        assert s_obj.tobytes() == g_obj[s0:s1].tobytes(), f"rank {r} objectives"
        assert s_acc.tobytes() == g_acc[s0:s1].tobytes(), f"rank {r} accumulators"
        # sampled solutions of this shard against the oracle (first, one forced fold, last)
        for k in sorted({s0 + 1, s0 + 7 + 16 * (r % 3), s1 - 1}):
            o_obj, o_acc = orc.eval(w.offsets[k])
            _assert_acc(g_acc[k], o_acc, f"C5 sol {k}")
            if o_acc.folds == 0:
                _assert_obj(g_obj[k], o_obj, f"C5 sol {k}")
            checked.append(k)
    assert len(checked) >= 3 * G - 2
    # fold flags and counts: bit-exact for every one of the 4096 solutions
    cnt = np.zeros(w.P, np.int32)
    sev = np.zeros(w.P, np.float64)
    flags = np.zeros((w.P, 2, w.T), np.uint8)
    ctx.check_folds(w.offsets, cnt, sev, flags)
    n_folded = 0
    for k in range(w.P):
        o_cnt, o_sev, o_flags = orc.check_folds(w.offsets[k])
        assert cnt[k] == o_cnt, k
        np.testing.assert_array_equal(flags[k], o_flags, err_msg=f"sol {k}")
        assert sev[k] == pytest.approx(o_sev, rel=1e-12, abs=1e-12)
        n_folded += o_cnt > 0
    assert n_folded >= w.P // 16  # the k = 7 (mod 16) forced folds are present
    unf = cnt == 0
    assert (g_acc["n_samples"][unf] == 2 * w.V).all()


@pytest.mark.parametrize("kind", ["class", "edges4", "edges16", "wholeclass", "all"])
def test_c4_partial_fos_size_sweep(wl, kind):
    w = wl(4)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    plan = fos_plan(w.tets, w.N)
    _, _, tc, off, acc = _gpu_full(ctx, w.offsets, cache=True)
    go, ch, nv = partial_request(w, plan, kind, 0)
    G = len(go) - 1
    nvd = torch.from_numpy(nv).to(DEV)
    outs = []
    for cache in (torch.from_numpy(tc).to(DEV), None):
        pobj = torch.empty((w.P * G, 3), dtype=torch.float64, device=DEV)
        pacc = torch.empty((w.P * G, 6), dtype=torch.int64, device=DEV)
        ctx.eval_partial(off, acc, go, ch, nvd, cache, pobj, pacc)
        torch.cuda.synchronize()
        outs.append((pobj.cpu().numpy(), morea.acc_to_numpy(pacc)))
    # cached == stateless, bitwise
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    assert outs[0][1].tobytes() == outs[1][1].tobytes()
    p_obj, p_acc = outs[0]
    groups = sorted({0, G // 2, G - 1})
    for k in (3, 200, w.P - 2):
        _, base_o = orc.eval(w.offsets[k])
        for g in groups:
            S = ch[go[g]:go[g + 1]]
            o_obj, o_acc = orc.eval_partial(w.offsets[k], base_o, S, nv[k, go[g]:go[g + 1]])
            _assert_acc(p_acc[k * G + g], o_acc, f"C4 {kind} sol {k} group {g}")
            if o_acc.folds == 0:
                _assert_obj(p_obj[k * G + g], o_obj, f"C4 {kind} sol {k} group {g}")

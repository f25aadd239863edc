"""GPU parity of the device-side optimal mixing of a colour class (NEXT-3,
PAPER.md §3; readings M1..M7 in DESIGN.md §3) against the CPU oracle
(run with -m gpu).  Sampled offsets are bit-exact; acceptance flags equal; the
final objectives within 1e-5; the carried state equals a fresh full evaluation."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.oracle import Acc, Oracle  # noqa: E402
from paper_2303_04873_b200 import morea  # noqa: E402
from tests.test_gpu_parity import DEV, _ctx, _gpu_full  # noqa: E402
from tests.test_oracle_mix import _class, model_from_population  # noqa: E402


def _acc_struct(a):
    s = Acc()
    for k in ("h_sum", "g_sum", "m_sum", "severity", "n_samples", "folds", "flags"):
        setattr(s, k, a[k].item() if hasattr(a[k], "item") else a[k])
    return s


@pytest.mark.parametrize("idx,P,nclu", [(1, 8, 1), (2, 16, 2)])
def test_mix_class_parity(wl, idx, P, nclu):
    w = wl(idx)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    go, ch = _class(w)
    offs = np.ascontiguousarray(w.offsets[:P])
    cluster = (np.arange(P) % nclu).astype(np.int32)
    models = [model_from_population(offs[cluster == c], go, ch, eps=0.01) for c in range(nclu)]
    mu = np.concatenate([m[0] for m in models])
    L = np.concatenate([m[1] for m in models])
    obj, acc, tc, off_d, acc_d = _gpu_full(ctx, offs, cache=True)
    archive = obj[[0, 2, 4]].copy()
    obj_d = torch.from_numpy(obj).to(DEV)
    tc_d = torch.from_numpy(tc).to(DEV)
    accepted = torch.zeros((P, len(go) - 1), dtype=torch.uint8, device=DEV)
    seed, gen, base = 77, 3, 100
    ctx.mix_class(off_d, acc_d, obj_d, tc_d, go, ch, cluster, mu, L, w.fixed_axes, archive, 0.0, seed, gen,
                  base, accepted)
    torch.cuda.synchronize()
    g_off = off_d.cpu().numpy()
    g_obj = obj_d.cpu().numpy()
    g_acc = morea.acc_to_numpy(acc_d)
    g_flags = accepted.cpu().numpy()
    assert g_flags.sum() > 0
    stride = 6 * len(ch)
    for k in range(P):
        c = cluster[k]
        assert np.array_equal(mu[c * stride:(c + 1) * stride], models[c][0])
        new, nacc, nobj, flags = orc.mix(offs[k], _acc_struct(acc[k]), obj[k], go, ch, models[c][0],
                                         models[c][1], w.fixed_axes, archive, 0.0, seed, gen, base + k)
        assert np.array_equal(flags, g_flags[k]), k
        assert np.array_equal(new.view(np.uint32), g_off[k].view(np.uint32)), k
        np.testing.assert_allclose(g_obj[k], nobj, rtol=1e-5, atol=1e-12)
        assert g_acc[k]["n_samples"] == nacc.n_samples and g_acc[k]["folds"] == nacc.folds
    # the carried state equals a fresh full evaluation of the new offsets
    f_obj, f_acc, f_tc, _, _ = _gpu_full(ctx, g_off, cache=True)
    np.testing.assert_allclose(g_obj, f_obj, rtol=1e-9)
    assert np.array_equal(g_acc["n_samples"], f_acc["n_samples"])
    assert np.array_equal(tc_d.cpu().numpy(), f_tc)

"""GPU parity of the batched fold repair (NEXT-2, §4.3.1;
readings P1..P8 in DESIGN.md §3) against the CPU oracle (run with -m gpu).

Bar: bit-exact.  Candidate draws, sigma, scores and the written offsets follow
the oracle's exact operation sequence, so the repaired offsets and the
moved / aborted counts must be identical.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.oracle import Oracle  # noqa: E402
from tests.test_gpu_parity import DEV, _ctx  # noqa: E402

SEED = 2024


def _gpu_repair(ctx, offsets, fixed, sol_base=0, host=False):
    P = offsets.shape[0]
    if host:
        off = np.ascontiguousarray(offsets, np.float32).copy()
        mv = np.zeros(P, np.int32)
        ab = np.zeros(P, np.int32)
        ctx.repair(off, SEED, fixed, sol_base, mv, ab)
        return off, mv, ab
    off = torch.from_numpy(np.ascontiguousarray(offsets, np.float32)).to(DEV)
    fx = torch.from_numpy(np.ascontiguousarray(fixed, np.uint8)).to(DEV)
    mv = torch.zeros(P, dtype=torch.int32, device=DEV)
    ab = torch.zeros(P, dtype=torch.int32, device=DEV)
    ctx.repair(off, SEED, fx, sol_base, mv, ab)
    torch.cuda.synchronize()
    return off.cpu().numpy(), mv.cpu().numpy(), ab.cpu().numpy()


def _heavy(w, scale, seed):
    """More folds: the workload's offsets with extra interior noise."""
    rng = np.random.default_rng(seed)
    fx6 = np.concatenate([w.fixed_axes, w.fixed_axes], 1)
    noise = rng.normal(0, scale, size=w.offsets.shape).astype(np.float32)
    return np.where(fx6[None], w.offsets, w.offsets + noise).astype(np.float32)


@pytest.mark.parametrize("idx", [1, 2])
def test_repair_bitexact_workload(wl, idx):
    w = wl(idx)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    offs = w.offsets if idx == 1 else _heavy(w, 5.0, 3)[:24]
    new, mv, ab = _gpu_repair(ctx, offs, w.fixed_axes)
    n_moved = 0
    for k in range(offs.shape[0]):
        o_new, o_mv, o_ab = orc.repair(offs[k], SEED, k, w.fixed_axes)
        assert np.array_equal(new[k].view(np.uint32), o_new.view(np.uint32)), k
        assert (mv[k], ab[k]) == (o_mv, o_ab), k
        n_moved += o_mv
    assert n_moved > 0  # the comparison is not vacuous


def test_repair_reduces_folds_and_sharding(wl):
    w = wl(2)
    ctx = _ctx(w)
    offs = _heavy(w, 5.0, 5)[:32]
    new, mv, ab = _gpu_repair(ctx, offs, w.fixed_axes)
    # sol_base keys the generator by global solution index: a shard reproduces its rows
    part, mv2, ab2 = _gpu_repair(ctx, offs[8:16], w.fixed_axes, sol_base=8)
    assert np.array_equal(part, new[8:16]) and np.array_equal(mv2, mv[8:16])
    # host buffers give the same result
    hnew, hmv, hab = _gpu_repair(ctx, offs[:8], w.fixed_axes, host=True)
    assert np.array_equal(hnew, new[:8]) and np.array_equal(hmv, mv[:8]) and np.array_equal(hab, ab[:8])
    # folds never increase (device fold check)
    c0 = torch.empty(32, dtype=torch.int32, device=DEV)
    s0 = torch.empty(32, dtype=torch.float64, device=DEV)
    c1 = torch.empty(32, dtype=torch.int32, device=DEV)
    s1 = torch.empty(32, dtype=torch.float64, device=DEV)
    ctx.check_folds(torch.from_numpy(offs).to(DEV), c0, s0)
    ctx.check_folds(torch.from_numpy(new).to(DEV), c1, s1)
    torch.cuda.synchronize()
    c0, s0, c1, s1 = (x.cpu().numpy() for x in (c0, s0, c1, s1))
    assert (c0 > 0).sum() > 4
    assert np.all((c1 < c0) | ((c1 == c0) & (s1 <= s0 + 1e-9)))
    assert c1.sum() < c0.sum()

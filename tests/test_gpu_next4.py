"""GPU parity of the rasterizer exports (NEXT-4: object counts and elasticity
factors, App. A.1; DVF export, §5.4; readings E1..E3 in
DESIGN.md §3) against the CPU oracle (run with -m gpu).  Bar: bit-exact (counts,
factors and the fp32 displacement field from the exact numerator)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)

from oracle.oracle import Oracle  # noqa: E402
from tests.test_gpu_parity import _ctx  # noqa: E402
from tests.test_oracle_next4 import _masks  # noqa: E402


@pytest.mark.parametrize("idx", [1, 2])
def test_label_counts_and_elasticity_bitexact(wl, idx):
    w = wl(idx)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    masks = _masks(w.dims, 7)
    for k, side in ((None, 0), (3, 0), (3, 1), (7, 1)):
        off = None if k is None else w.offsets[k]
        g = ctx.label_counts(off, side, masks, 3)
        o = orc.label_counts(off, side, masks, 3)
        assert np.array_equal(g, o), (k, side)
    f = [10.0, 0.5, 2.0]
    assert np.array_equal(ctx.elasticity(masks, f).view(np.uint32), orc.elasticity(masks, f).view(np.uint32))


@pytest.mark.parametrize("idx,k", [(1, 2), (2, 3), (2, 7)])
def test_dvf_bitexact(wl, idx, k):
    w = wl(idx)
    ctx = _ctx(w)
    orc = Oracle.from_workload(w)
    for side in (0, 1):
        gd, gc = ctx.dvf(w.offsets[k], side)
        od, oc = orc.dvf(w.offsets[k], side)
        assert np.array_equal(gc, oc), side
        assert np.array_equal(gd.view(np.uint32), od.view(np.uint32)), side
    # device buffers give the same field
    off = torch.from_numpy(np.ascontiguousarray(w.offsets[k])).cuda()
    dd = torch.empty((w.V, 3), dtype=torch.float32, device="cuda")
    dc = torch.empty(w.V, dtype=torch.uint8, device="cuda")
    ctx.dvf(off, 1, dd, dc)
    torch.cuda.synchronize()
    assert np.array_equal(dd.cpu().numpy(), gd) and np.array_equal(dc.cpu().numpy(), gc)

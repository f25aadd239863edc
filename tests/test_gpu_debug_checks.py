"""Device-side checks over every kernel family (run with -m gpu).

compute-sanitizer is closed on the GPU pool this round was built on ("runs under it
have left GPUs needing a reset").  In its place the library is built a second time
with -DMOREA_DEBUG_CHECKS (libmorea_debug.so): MOREA_CHECK asserts on the device
check the indices of the shared-memory row tables, row-start bitmap windows,
slice tables and guidance queue of k_raster, the own-record and footprint ranges
of every sample, the offset / new-value slots of every tet, and the queue's item
decoding.  tools/checks_target.py drives full, cached and stateless partial,
fold check, owner map, sample-map dump, Sobol, repair, exports and optimal mixing
on C1 and C2 through the C-ABI; a failed check traps the kernel (non-zero exit).
The outputs of the checked build must be bitwise equal to the release build's.
"""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2303_04873_b200")


def _run(lib, cfg):
    env = dict(os.environ, MOREA_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "checks_target.py"), str(cfg)],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, (lib, r.stdout[-2000:] + r.stderr[-4000:])
    assert "checks target ok" in r.stdout
    return json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])


@pytest.mark.parametrize("cfg", [1, 2])
def test_device_checks_clean_and_bitwise_equal(cfg):
    from paper_2303_04873_b200 import build
    dbg = build.build_debug()
    a = _run(os.path.join(PKG, "libmorea.so"), cfg)
    b = _run(dbg, cfg)
    assert a == b

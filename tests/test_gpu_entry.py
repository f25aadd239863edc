"""The driver's entry points on a real GPU (run with -m gpu): smoke() runs the C1
full + partial evaluation through the C-ABI on cuda:0 and checks it against the
oracle; the library it loads must be the in-tree libmorea.so (no fallback)."""
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)


def test_smoke_entry():
    import __graft_entry__
    __graft_entry__.smoke()


def test_loaded_library_is_in_tree():
    from paper_2303_04873_b200 import morea
    if os.environ.get("MOREA_LIB"):
        pytest.skip("MOREA_LIB overrides the library (dev A/B runs)")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    want = os.path.realpath(os.path.join(root, "paper_2303_04873_b200", "libmorea.so"))
    maps = open("/proc/self/maps").read()
    assert want in maps, "libmorea.so from the repo is not mapped into this process"
    assert os.path.realpath(morea.LIB_PATH) == want

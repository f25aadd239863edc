"""CPU-side checks of the C-ABI library (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "morea.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(morea_[a-z_]+)\s*\(", src)))


def test_header_declares_the_five_calls():
    names = _declared()
    for n in ("morea_load_images", "morea_set_mesh", "morea_eval_full", "morea_eval_partial",
              "morea_check_folds"):
        assert n in names


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2303_04873_b200 import build, morea
    build.build()
    lib = ctypes.CDLL(morea.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    assert sorted(morea.EXPORTS) == _declared()


def test_acc_layout_matches_header():
    """morea_acc is 4 doubles, int64, 2 x int32 = 48 bytes (include/morea.h)."""
    from paper_2303_04873_b200 import morea
    assert morea.ACC_DTYPE.itemsize == 48
    assert list(morea.ACC_DTYPE.names) == ["h_sum", "g_sum", "m_sum", "severity", "n_samples",
                                          "folds", "flags"]


def test_create_without_gpu_fails_cleanly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2303_04873_b200 import morea
    with pytest.raises(morea.MoreaError):
        morea.Context(0)


def test_no_oracle_import_in_product():
    """The product package never imports or links the oracle (parity independence)."""
    pkg = os.path.join(ROOT, "paper_2303_04873_b200")
    pat = re.compile(r"(import\s+oracle|from\s+oracle|liboracle|morea_oracle|#include\s+\"[^\"]*oracle)")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not pat.search(txt), f

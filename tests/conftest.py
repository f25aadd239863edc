import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger configuration (C3/C4)")


_WL = {}


def workload(idx, P=None):
    """Cached synthetic workload (generation is deterministic and seeded)."""
    from synth import make_workload
    key = (idx, P)
    if key not in _WL:
        _WL[key] = make_workload(idx, P=P)
    return _WL[key]


@pytest.fixture(scope="session")
def wl():
    return workload

"""The N > 1 path of bench.py run for real (run with -m gpu).

The test boxes have one GPU, so two ranks share it through the gloo backend
(`--dist-backend gloo`: per-solution records staged through host memory).  Each
rank evaluates its contiguous block of the C4 population (256 of 512
solutions), the records of the full evaluation and of every colour class's
partial evaluation are all-gathered, and the step time is the max over ranks.
The gathered records must be bitwise equal to a single-rank run over the same
512 solutions (no cross-rank arithmetic, fixed summation order).  The driver's
8-GPU run keeps NCCL, the default backend.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_line(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_two_ranks_gloo_equals_one_rank(tmp_path):
    one, two = str(tmp_path / "one.npy"), str(tmp_path / "two.npy")
    common = ["--steps", "2", "--warmup", "3", "--quick"]
    r1 = subprocess.run([sys.executable, "bench.py", *common, "--pop-per-rank", "512", "--dump-records", one],
                        cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r1.returncode == 0, r1.stderr[-3000:]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    r2 = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                         "--master-addr", "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2",
                         *common, "--pop-per-rank", "256", "--dist-backend", "gloo", "--dump-records", two],
                        cwd=ROOT, capture_output=True, text=True, timeout=1200, env=env)
    assert r2.returncode == 0, r2.stderr[-3000:]
    j1, j2 = _json_line(r1.stdout), _json_line(r2.stdout)
    assert j1["n_gpus"] == 1 and j2["n_gpus"] == 2
    assert j1["config"]["population_total"] == j2["config"]["population_total"] == 512
    a, b = np.load(one), np.load(two)
    assert a.shape == b.shape and a.dtype == b.dtype == np.int64
    assert np.array_equal(a, b)
    assert j2["value"] > 0 and j2["ms_per_step"] > 0

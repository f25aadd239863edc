"""The NCCL leg of the population all-gather (row a10) on a real GPU (run with -m gpu).

Only one GPU is available to the tests, so this runs a world of one rank over
NCCL: the records of a C2 full and partial evaluation go through
all_gather_into_tensor on the context stream and must come back bitwise.
The multi-rank gather logic (padding, shard order) is covered on CPU by the
world-2 gloo tests (tests/test_distributed_gloo.py).
"""
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # collected on CPU boxes, skipped there
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402

from paper_2303_04873_b200.distributed import all_gather_records, pack, unpack  # noqa: E402
from synth import fos_plan, partial_request  # noqa: E402
from tests.test_gpu_parity import DEV, _ctx, _gpu_full  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_nccl_all_gather_world_one(wl):
    w = wl(2)
    ctx = _ctx(w)
    obj, acc, tc, off, acc_d = _gpu_full(ctx, w.offsets, cache=True)
    plan = fos_plan(w.tets, w.N)
    go, ch, nv = partial_request(w, plan, "class", 0)
    G = len(go) - 1
    pobj = torch.empty((w.P * G, 3), dtype=torch.float64, device=DEV)
    pacc = torch.empty((w.P * G, 6), dtype=torch.int64, device=DEV)
    ctx.eval_partial(off, acc_d, go, ch, torch.from_numpy(nv).to(DEV), torch.from_numpy(tc).to(DEV), pobj, pacc)
    torch.cuda.synchronize()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1,
                            device_id=DEV)
    try:
        stream = torch.cuda.ExternalStream(ctx.stream_handle, device=DEV)
        obj_d = torch.from_numpy(obj).to(DEV)
        with torch.cuda.stream(stream):
            full = all_gather_records(pack(obj_d, acc_d), w.P)
            part = all_gather_records(pack(pobj, pacc), w.P, rows_per_solution=G)
        torch.cuda.synchronize()
        assert dist.get_backend() == "nccl"
    finally:
        dist.destroy_process_group()
    f_obj, f_acc = unpack(full)
    assert np.array_equal(f_obj.cpu().numpy(), obj)
    assert f_acc.cpu().numpy().tobytes() == acc_d.cpu().numpy().tobytes()
    p_obj, p_acc = unpack(part)
    assert p_obj.cpu().numpy().tobytes() == pobj.cpu().numpy().tobytes()
    assert p_acc.cpu().numpy().tobytes() == pacc.cpu().numpy().tobytes()

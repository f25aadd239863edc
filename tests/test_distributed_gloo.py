"""world_size-2 gloo tests of the population-sharding path (row a10) on CPU.

Each rank evaluates its contiguous block of solutions (here with the oracle,
since there is no GPU on the CPU box) and the per-solution records are
all-gathered with paper_2303_04873_b200.distributed; the gathered result must be
bitwise equal to evaluating the whole population in one process.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2303_04873_b200.distributed import (RECORD_WORDS, all_gather_records, pack,
                                               shard_bounds, unpack)


def _records(w, sols, plan_req=None):
    from oracle.oracle import Oracle
    orc = Oracle.from_workload(w)
    obj, acc = [], []
    for k in sols:
        o, a = orc.eval(w.offsets[k])
        obj.append(o)
        acc.append(np.frombuffer(bytes(a), dtype=np.int64))
        if plan_req is not None:
            go, ch, nv = plan_req
            for g in range(len(go) - 1):
                po, pa = orc.eval_partial(w.offsets[k], a, ch[go[g]:go[g + 1]], nv[k, go[g]:go[g + 1]])
                obj.append(po)
                acc.append(np.frombuffer(bytes(pa), dtype=np.int64))
    return (torch.tensor(np.array(obj), dtype=torch.float64),
            torch.tensor(np.array(acc), dtype=torch.int64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, P_total, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from synth import fos_plan, make_workload, partial_request
    w = make_workload(1, P=P_total)
    plan = fos_plan(w.tets, w.N)
    req = partial_request(w, plan, "class", 0)
    G = len(req[0]) - 1
    s0, s1 = shard_bounds(P_total, world, rank)
    obj, acc = _records(w, range(s0, s1), req)
    full = all_gather_records(pack(obj, acc), P_total, rows_per_solution=1 + G)
    if rank == 0:
        out_q.put(full.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("P_total", [8, 7])
def test_gloo_world2_allgather_equals_single_process(P_total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, P_total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from synth import fos_plan, make_workload, partial_request
    w = make_workload(1, P=P_total)
    plan = fos_plan(w.tets, w.N)
    req = partial_request(w, plan, "class", 0)
    obj, acc = _records(w, range(P_total), req)
    ref = pack(obj, acc).numpy()
    assert got.shape == ref.shape == (P_total * (len(req[0])), RECORD_WORDS)
    assert got.tobytes() == ref.tobytes()
    o2, a2 = unpack(torch.from_numpy(got))
    assert torch.equal(o2.nan_to_num(-1), obj.nan_to_num(-1)) and torch.equal(a2, acc)


def test_shard_bounds_cover_exactly_once():
    for P in (1, 7, 512, 4096, 4097):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(P, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == P
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1

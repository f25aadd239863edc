"""Population sharding across ranks.

Solutions are independent, so the population is split into contiguous blocks,
one per rank (one process per GPU); every rank holds full replicas of the
volumes, maps and mesh (one morea Context each).  After a rank evaluated its
block, the per-solution outputs (3 objectives + the 48-byte accumulator per
solution and group) are all-gathered -- over NCCL/NVLink on GPUs, gloo on CPU.
There is no cross-rank arithmetic, so G-rank outputs are bitwise equal to a
single-rank evaluation.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

# per solution x group: obj (3 x f64) + morea_acc (48 B = 6 x i64) = 9 x 8 bytes
RECORD_WORDS = 9


def shard_bounds(P_total: int, world: int, rank: int):
    """Contiguous block [start, stop) of rank `rank`; blocks differ by <= 1 solution."""
    base, extra = divmod(P_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def pack(obj: torch.Tensor, acc: torch.Tensor) -> torch.Tensor:
    """(P*G, 3) f64 objectives + (P*G, 6) i64 accumulators -> (P*G, 9) i64 records."""
    return torch.cat([obj.contiguous().view(torch.int64), acc.contiguous()], dim=1)


def unpack(rec: torch.Tensor):
    return rec[:, :3].contiguous().view(torch.float64), rec[:, 3:].contiguous()


def all_gather_records(local: torch.Tensor, P_total: int, rows_per_solution: int = 1,
                       group=None) -> torch.Tensor:
    """All-gather the (P_local*rows, 9) int64 records of every rank into (P_total*rows, 9).

    Blocks are padded to the largest shard so one all_gather_into_tensor (NCCL)
    moves everything; padding rows are dropped afterwards.
    """
    world = dist.get_world_size(group)
    rows_max = (P_total + world - 1) // world * rows_per_solution
    nccl = dist.get_backend(group) == "nccl"
    # gloo moves host tensors: device records are staged through host memory
    dev = local.device if nccl else torch.device("cpu")
    buf = torch.zeros((rows_max, RECORD_WORDS), dtype=torch.int64, device=dev)
    buf[: local.shape[0]] = local.to(dev)
    out = torch.empty((world * rows_max, RECORD_WORDS), dtype=torch.int64, device=dev)
    if nccl:
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        parts = list(out.chunk(world))
        dist.all_gather(parts, buf, group=group)
        out = torch.cat(parts)
    keep = []
    for r in range(world):
        s, e = shard_bounds(P_total, world, r)
        keep.append(out[r * rows_max: r * rows_max + (e - s) * rows_per_solution])
    return torch.cat(keep).to(local.device)

"""Environment sharding across GPUs (one process per GPU).

The reference's only parallelism is data parallelism over environments:
chunked contiguous ranges per std::thread, every env writing only its own
slot, results independent of worker count (src/batch.cpp:26-41, 207-215).
Across GPUs the same holds: contiguous env ranges, no collective on the hot
path; an optional end-of-run gather of the per-env reduced result
(mean_contact_distance, 4 B/env) over torch.distributed (NCCL over NVLink on
the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple


def shard_range(n_total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) of rank's envs; sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard_range: need 0 <= rank < world")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def gather_shards(local, n_total: int, rank: int, world: int, group=None):
    """All-gather per-env results (1-D tensor of this rank's shard) into the
    full [n_total] tensor on every rank, padding uneven shards."""
    import torch
    import torch.distributed as dist

    lo, hi = shard_range(n_total, rank, world)
    width = shard_range(n_total, 0, world)[1]  # rank 0 has the largest shard
    buf = torch.zeros(width, dtype=local.dtype, device=local.device)
    buf[: hi - lo] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = []
    for r in range(world):
        a, b = shard_range(n_total, r, world)
        out.append(parts[r][: b - a])
    return torch.cat(out)


def run_sharded(compute: Callable[[int, int], "object"], n_total: int, rank: int, world: int,
                gather: bool = True, group=None):
    """compute(lo, hi) -> per-env results of this shard; optionally gathered."""
    lo, hi = shard_range(n_total, rank, world)
    local = compute(lo, hi)
    if not gather or world == 1:
        return local
    return gather_shards(local, n_total, rank, world, group)

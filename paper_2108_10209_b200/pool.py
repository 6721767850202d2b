"""Multi-GPU sharding of independent images.

Images share nothing, so the data path has no collective: one process per GPU
(torchrun), each with its own engine context.  Work is handed out through the
torch.distributed key-value store (TCPStore `add` is an atomic counter): a
dynamic queue like the reference CLI's process pool (cli.py:207-211), which
absorbs the per-image imbalance of early stopping.  The only collectives are
host-side bookkeeping over a gloo group on CPU tensors (north_star (4): no
NCCL): a barrier before/after the timed region and a MAX reduction of the
per-rank device times.
"""

from __future__ import annotations

import os
from typing import Iterator


def dist_env() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def default_store():
    import torch.distributed as dist

    if not dist.is_initialized():
        return None
    return dist.distributed_c10d._get_default_store()


def claim(store, key: str, total: int) -> Iterator[int]:
    """Yield image indices this rank claims from a shared counter until the
    queue is empty.  Without a store (single process) yields 0..total-1."""
    if store is None:
        yield from range(total)
        return
    while True:
        i = int(store.add(key, 1)) - 1
        if i >= total:
            return
        yield i


def static_shard(total: int, rank: int, world: int) -> list[int]:
    """Round-robin split (deterministic fallback when no store is available)."""
    return list(range(rank, total, world))


def max_over_ranks(value: float, device=None) -> float:
    """MAX of a per-rank scalar (device time) across the job."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_over_ranks(value: float, device=None) -> list[float]:
    """Every rank's scalar (e.g. per-GPU busy time), in rank order."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(value)]
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [float(x.item()) for x in out]


def imbalance(busy: list[float]) -> float:
    """max / mean of the per-rank busy times (1.0 = perfectly balanced)."""
    mean = sum(busy) / len(busy)
    return max(busy) / mean if mean > 0 else 1.0

"""Multi-GPU plumbing for the streaming configs.

Records are independent, so N ranks take N disjoint contiguous shards of the
seeded stream and never exchange data; the only collectives are the timing
barrier and the max-over-ranks of the measured time.
"""
from __future__ import annotations


def shard(rank: int, world: int, n_total: int) -> tuple[int, int]:
    """(first, count) of rank's contiguous share of n_total records."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = n_total * rank // world
    hi = n_total * (rank + 1) // world
    return lo, hi - lo


def weak_shard(rank: int, n_per_rank: int) -> tuple[int, int]:
    """Weak scaling: every rank owns n_per_rank records of the global stream."""
    return rank * n_per_rank, n_per_rank


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (elapsed time) over the process group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())

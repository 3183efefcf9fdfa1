"""Multi-GPU host logic: the path shards by image with no data-path collective.

Weak scaling: with a per-GPU batch B, rank r of N transforms the global images [r*B, (r+1)*B); the
only collective is the max over ranks of the measured step time (the job is as slow as its
slowest GPU). Pure torch.distributed plumbing, usable with nccl (bench) or gloo (CPU tests).
"""
from __future__ import annotations


def rank_images(per_rank: int, rank: int, world: int) -> range:
    """Global image indices owned by `rank` (weak scaling: every rank owns `per_rank` images)."""
    if per_rank < 1 or world < 1 or not 0 <= rank < world:
        raise ValueError("bad shard request")
    return range(rank * per_rank, (rank + 1) * per_rank)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar over the default process group (identity when not initialised)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())

"""Multi-GPU plumbing of the rollout: prompt sharding and step statistics.

Rollout shards by prompt exactly like the reference assigns requests to
worker groups -- request ``i`` goes to worker ``i mod n`` (``sim.py:307-309``)
-- so every rank runs an independent rollout of its shard (weak scaling, no
data-path collective).  Ranks only meet to time the step: the job's time is
the max over ranks, its committed tokens the sum (``torch.distributed``;
NCCL on GPUs, gloo in CPU tests).
"""

from __future__ import annotations


def shard(items: list, rank: int, world: int) -> list:
    """Round-robin prompt sharding (``sim.py:307-309``)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    return items[rank::world]


def reduce_step_stats(elapsed_ms: list[float], committed: list[float], dist=None, device="cpu"):
    """(max over ranks of each elapsed time, sum over ranks of each count)."""
    import torch

    t = torch.tensor(elapsed_ms, dtype=torch.float64, device=device)
    c = torch.tensor(committed, dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return t.tolist(), c.tolist()

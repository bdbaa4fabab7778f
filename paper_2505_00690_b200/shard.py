"""Env sharding across ranks: one process per GPU, rank r of W
owns the contiguous global env ids [r*E, (r+1)*E).  Envs never exchange data
(SPEC: no cross-environment sharing; every per-env stream derives from the
global env id, batch.py:85), so the data path has no collective; the only one
is an all_gather of per-env stats at the end of a run.
"""

import numpy as np

from .rng import child_seed

STAT_FIELDS = ("last_gap", "objects", "walkable", "active_agents", "steps", "status")


def env_ids(rank, world, per_rank):
    """Global env ids owned by ``rank`` (weak scaling: ``per_rank`` envs each)."""
    if not (0 <= rank < world):
        raise ValueError("rank outside [0, world)")
    return np.arange(rank * per_rank, (rank + 1) * per_rank, dtype=np.int64)


def env_seeds(master_seed, ids):
    """child_seed(master, "env", global_id) -- identical whatever the sharding."""
    return [child_seed(master_seed, "env", int(i)) for i in ids]


def gather_env_stats(stats, group=None):
    """all_gather (E_local, F) per-env stats into (W*E_local, F) on every rank,
    ordered by rank (= by global env id).  Works with NCCL (device tensors) and
    gloo (CPU tensors)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return stats
    world = dist.get_world_size(group)
    out = [torch.empty_like(stats) for _ in range(world)]
    dist.all_gather(out, stats.contiguous(), group=group)
    return torch.cat(out, 0)


def max_over_ranks(value, device=None, group=None):
    """Max of a scalar over ranks (the timing rule: max over ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())

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
    dev = stats.device
    if dist.get_backend(group) == "gloo" and dev.type != "cpu":
        stats = stats.cpu()         # gloo gathers host tensors
    out = [torch.empty_like(stats) for _ in range(world)]
    dist.all_gather(out, stats.contiguous(), group=group)
    return torch.cat(out, 0).to(dev)


def max_over_ranks(value, device=None, group=None):
    """Max of a scalar over ranks (the timing rule: max over ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return float(value)
    if dist.get_backend(group) == "gloo":
        device = "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def max_tensor_over_ranks(t, group=None):
    """Elementwise max of a float64 tensor over ranks (NCCL device / gloo host)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return t
    dev = t.device
    if dist.get_backend(group) == "gloo" and dev.type != "cpu":
        t = t.cpu()
    t = t.clone()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.to(dev)


_P = 2147483647   # 2^31 - 1: every product below stays < 2^62, every row sum < 2^63


def _weighted_mod(words):
    """Two position-weighted sums mod P over the columns of (R, n) int64 words < P."""
    import torch
    k = torch.arange(words.shape[1], dtype=torch.int64, device=words.device)
    w1 = (k * 40503 + 1) % _P
    w2 = (k * 69069 + 12345) % _P
    s1 = ((words * w1) % _P).sum(1) % _P
    s2 = ((words * w2) % _P).sum(1) % _P
    return s1 * _P + s2


def state_checksum(*arrays):
    """Per-env checksum of float64 state arrays shaped (E, ...): the exact bit
    patterns, position-weighted, reduced mod 2^31 - 1 (two independent sums,
    an int64 < 2^62 per env).  Integer arithmetic only, so the value is the same
    on any device and for any sharding of the envs."""
    import torch
    as_t = lambda a: a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))   # state views: one copy
    parts = [as_t(a).reshape(a.shape[0], -1).to(torch.float64) for a in arrays]
    x = torch.cat(parts, 1).contiguous().view(torch.int64)
    words = torch.stack([x & 0xFFFFFFFF, (x >> 32) & 0xFFFFFFFF], 2).reshape(x.shape[0], -1) % _P
    return _weighted_mod(words)


def checksum_of(checksums):
    """Checksum of per-env checksums (in global env order) -> python int."""
    import torch
    c = torch.as_tensor(checksums).reshape(1, -1).to(torch.int64)
    words = torch.stack([c % _P, c // _P], 2).reshape(1, -1)
    return int(_weighted_mod(words)[0])

"""Seed tree (src/rng.py:15-26): host child_seed plus the batched device form."""

import hashlib

import numpy as np

from . import _lib

_MASK64 = (1 << 64) - 1
LABEL_IDS = {"env": 0, "crowd-run": 1, "crowd": 2, "resample": 3}


def child_seed(parent, *labels):
    """rng.py:15-19 (host; used for single seeds)."""
    key = str(int(parent) & _MASK64) + "".join(f":{l}" for l in labels)
    return int.from_bytes(hashlib.sha256(key.encode("utf-8")).digest()[:8], "little")


def child_seeds_device(parents, label, k=None, stream=None):
    """child_seed(parents[i], label[, k[i]]) for a device int64 tensor of parents."""
    import torch
    parents = parents.to(torch.int64).contiguous()
    out = torch.empty_like(parents)
    kk = None if k is None else torch.as_tensor(k, dtype=torch.int64, device=parents.device).expand_as(parents).contiguous()
    err = _lib.lib().cw_child_seeds(parents.numel(), _lib.ptr(parents), LABEL_IDS[label],
                                    _lib.ptr(kk), _lib.ptr(out), _lib.stream_ptr(stream))
    _lib.check(err, "cw_child_seeds")
    return out


def seeds_to_tensor(seeds, device):
    import torch
    arr = np.array([int(s) & _MASK64 for s in seeds], dtype=np.uint64).view(np.int64)
    return torch.from_numpy(arr).to(device)

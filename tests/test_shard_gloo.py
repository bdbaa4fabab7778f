"""N>1 path on CPU: world_size-2 gloo process group, the same sharding and
stats gather bench.py uses over NCCL.  The per-env results are
computed with the oracle (CPU) and must be invariant to the sharding."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_00690_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _per_env_stats(global_ids, catalog_path):
    """A small, sharding-invariant per-env computation: oracle scene + crowd ticks."""
    import json
    from oracle import crowd as C
    from oracle import scene as S
    from oracle.rng import child_seed
    cat = S.load_catalog_tuples(json.load(open(catalog_path)))
    mix = {"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}
    rows, sums = [], []
    for gid in global_ids:
        s = child_seed(0, "env", int(gid))
        sc = S.generate_scene(dict(seed=s, extent=(12.0, 12.0), res=0.25, task="NavDynamic",
                                   split="Train", density=1.0, mix=mix), cat)
        sp = C.spawn_agents(sc["labels"], 0.25, 3, child_seed(s, "crowd", 0))
        f = C.CrowdFieldOracle([(sc["labels"], 0.25)], C.Config(), [child_seed(s, "crowd-run")])
        f.set_agents([sp])
        for _ in range(3):
            f.step()
        rows.append([float(f.pos.sum()), float(f.vel.sum()), len(sc["objects"]),
                     float((sc["labels"] == 2).sum()), float(f.last_gap_by_env[0]), 3.0])
        sums.append(shard.state_checksum(f.pos, f.vel, f.goal)[0])
    return torch.tensor(rows, dtype=torch.float64), torch.stack(sums)


def _worker(rank, world, port, per_rank, catalog_path, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = shard.env_ids(rank, world, per_rank)
    local, csum = _per_env_stats(ids, catalog_path)
    full = shard.gather_env_stats(local)
    csum_full = shard.gather_env_stats(csum[:, None])[:, 0]
    t = shard.max_over_ranks(float(rank) + 0.5)
    if rank == 0:
        torch.save({"full": full, "csum": csum_full, "max": t}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_env_ids_partition():
    ids = [shard.env_ids(r, 4, 3) for r in range(4)]
    assert np.array_equal(np.concatenate(ids), np.arange(12))
    with pytest.raises(ValueError):
        shard.env_ids(4, 4, 3)
    assert shard.env_seeds(0, [5]) == shard.env_seeds(0, np.array([5]))


def test_two_rank_gloo_gather_matches_single_process(tmp_path):
    from conftest import GOLDEN
    cat = os.path.join(GOLDEN, "catalog.json")
    out = str(tmp_path / "gathered.pt")
    per_rank = 2
    mp.spawn(_worker, args=(2, _free_port(), per_rank, cat, out), nprocs=2, join=True)
    got = torch.load(out)
    ref, ref_sum = _per_env_stats(np.arange(2 * per_rank), cat)
    assert torch.equal(got["full"], ref)          # sharding-invariant, rank-ordered
    assert torch.equal(got["csum"], ref_sum)      # per-env state checksums, exact
    assert shard.checksum_of(got["csum"]) == shard.checksum_of(ref_sum)
    assert got["max"] == 1.5                      # max over ranks


def test_state_checksum_exact_and_shard_invariant():
    g = torch.Generator().manual_seed(5)
    pos = torch.randn(8, 7, 2, dtype=torch.float64, generator=g)
    vel = torch.randn(8, 7, 2, dtype=torch.float64, generator=g)
    c = shard.state_checksum(pos, vel)
    assert c.dtype == torch.int64 and c.shape == (8,)
    assert torch.equal(torch.cat([shard.state_checksum(pos[:3], vel[:3]),
                                  shard.state_checksum(pos[3:], vel[3:])]), c)
    assert torch.equal(shard.state_checksum(pos.numpy(), vel.numpy()), c)
    v2 = vel.clone()
    v2[5, 6, 1] = np.nextafter(v2[5, 6, 1].item(), np.inf)     # one ulp in one env
    c2 = shard.state_checksum(pos, v2)
    assert (c2 != c).tolist() == [False] * 5 + [True] + [False] * 2
    assert shard.checksum_of(c) != shard.checksum_of(c2)
    assert shard.checksum_of(c) != shard.checksum_of(c.flip(0))     # order matters
    z = torch.zeros(3, 4, dtype=torch.float64)
    assert not torch.equal(shard.state_checksum(z), shard.state_checksum(-z))   # bits, not values

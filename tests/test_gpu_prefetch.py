"""Next-tick search prefetch (cw_spec_create): CrowdField.step with the
prefetch must equal CrowdField.step without it bit for bit, tick after tick, while the
cache is actually used -- including when the predictions go stale: re-sampled grids
(cfg5's mix), per-tick env masks, caller writes into the state between ticks, and
replace_env with a host grid.  (Every other step() test, oracle parity included, runs
with the prefetch on: it is the default.)"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STATE = ("pos_t", "vel_t", "goal_t", "waypoint_t", "path_head_t", "path_n_t", "last_gap_t", "active_t")


def _setup(cfg, E):
    import torch
    import bench
    from paper_2505_00690_b200.rng import child_seeds_device
    from paper_2505_00690_b200.urbangen import SceneSampler
    bench.CFG.clear()
    bench.CFG.update(bench.CONFIGS[cfg])
    zero = torch.zeros(E, dtype=torch.int64, device="cuda")
    env = child_seeds_device(zero, "env", torch.arange(E, device="cuda"))
    s = SceneSampler(bench.make_spec(), E)
    s.sample(env, child_seeds_device(env, "crowd", 0))
    return s, env


def _fields(b, env, nd):
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
    from paper_2505_00690_b200.rng import child_seeds_device
    seeds = [int(x) for x in child_seeds_device(env, "crowd-run").cpu().numpy().view(np.uint64)]
    on = CrowdField(b, CrowdConfig(neighbor_distance=nd), seeds, prefetch=True)
    off = CrowdField(b, CrowdConfig(neighbor_distance=nd), seeds, prefetch=False)
    on.set_from_spawn(b)
    off.set_from_spawn(b)
    return on, off


def _robot(b, res, E, seed=7):
    import torch
    nx = b.labels.shape[2]
    g = torch.Generator(device="cpu").manual_seed(seed)
    pick = (torch.rand(E, generator=g).to("cuda") * b.walk_n.double()).long()
    cell = b.walk.gather(1, pick[:, None])[:, 0].long()
    rp = torch.stack([((cell % nx).double() + 0.5) * res, ((cell // nx).double() + 0.5) * res], 1).contiguous()
    return rp, torch.zeros_like(rp)


def _same(on, off, k):
    import torch
    for name in STATE:
        assert torch.equal(getattr(on, name), getattr(off, name)), (k, name)
    # the paths themselves (only the live part is meaningful)
    assert torch.equal(on.path_cells_t * (on.path_n_t[..., None] > 1), off.path_cells_t * (off.path_n_t[..., None] > 1)), k


@pytest.mark.parametrize("cfg,E,ticks", [("cfg2", 96, 60), ("cfg3", 48, 40)])
def test_prefetch_step_equals_plain_step(cfg, E, ticks, torch_cuda):
    import bench
    s, env = _setup(cfg, E)
    b = s.batch
    on, off = _fields(b, env, bench.CFG["nd"])
    rp, rv = _robot(b, float(b.params.res), E)
    for k in range(ticks):
        rp[:, 0] += 0.01   # the robot moves: only the ORCA half of a tick sees it
        on.step(rp, rv, 0.35)
        off.step(rp, rv, 0.35)
        _same(on, off, k)
    st = on.stats()
    assert st["prefetch_batches"] == ticks
    assert st["prefetch_hits"] > 0, st
    assert off.prefetch_stats() == {}


def test_prefetch_survives_stale_predictions(torch_cuda):
    """cfg5-style re-sampling between ticks, random env masks, caller writes into
    pos / goal, and replace_env: every prediction these invalidate must be ignored."""
    import torch
    import bench
    from paper_2505_00690_b200.rng import child_seeds_device
    E = 64
    s, env = _setup("cfg5", E)
    b = s.batch
    on, off = _fields(b, env, bench.CFG["nd"])
    res = float(b.params.res)
    rp, rv = _robot(b, res, E)
    rng = np.random.default_rng(3)
    counts = torch.zeros(E, dtype=torch.int64, device="cuda")
    for k in range(50):
        if k % 5 == 2:   # re-sample a few rows (new grids, new agents) in both fields
            rows = torch.from_numpy(rng.choice(E, 3, replace=False)).to("cuda")
            counts[rows] += 1
            s.sample(child_seeds_device(env[rows], "resample", counts[rows]),
                     child_seeds_device(env[rows], "crowd", counts[rows]), slots=rows)
            on.set_from_spawn(b, rows=rows)
            off.set_from_spawn(b, rows=rows)
        if k % 7 == 3:   # the caller moves a few agents (state views write through)
            e = int(rng.integers(E))
            for f in (on, off):
                f.pos[e, 0] = np.asarray(f.goal[e, 1])
        if k == 20:      # a host grid replaces env 5 in both fields
            occ = b.occupancy(int(rng.integers(E)))
            on.replace_env(5, occ)
            off.replace_env(5, occ)
        mask = None if k % 4 else (rng.random(E) < 0.7)
        on.step(rp, rv, 0.35, env_mask=mask)
        off.step(rp, rv, 0.35, env_mask=mask)
        _same(on, off, k)
    assert on.stats()["prefetch_hits"] > 0

"""Asynchronous scene sampling for per-tick re-sampling (envcore.SceneStandby): a reset
that installs the row's standby scene (sampled ahead on a side stream with the seeds the
reset would use) must leave exactly the state that re-sampling at the reset leaves --
scenes, route anchors, spawned crowds and the crowd ticks that follow."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCENE = ("labels", "elev", "nearest", "walk_n", "moves", "reach", "obj_pose", "obj_n", "routes", "n_routes",
         "sp_pos", "sp_goal", "scene_seed")
CROWD = ("pos_t", "vel_t", "goal_t", "waypoint_t", "path_n_t", "last_gap_t")


def _world(E):
    import torch
    import bench
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
    from paper_2505_00690_b200.rng import child_seeds_device
    from paper_2505_00690_b200.urbangen import SceneSampler
    bench.CFG.clear()
    bench.CFG.update(bench.CONFIGS["cfg5"])
    zero = torch.zeros(E, dtype=torch.int64, device="cuda")
    env = child_seeds_device(zero, "env", torch.arange(E, device="cuda"))
    s = SceneSampler(bench.make_spec(), E)
    s.sample(env, child_seeds_device(env, "crowd", 0))
    seeds = [int(x) for x in child_seeds_device(env, "crowd-run").cpu().numpy().view(np.uint64)]
    f = CrowdField(s.batch, CrowdConfig(neighbor_distance=bench.CFG["nd"]), seeds)
    f.set_from_spawn(s.batch)
    return s, f, env, torch.zeros(E, dtype=torch.int64, device="cuda")


@pytest.mark.parametrize("with_field", [False, True])
def test_standby_resets_equal_resampling(with_field, torch_cuda):
    """with_field: the standby crowds' first-tick searches are predicted on the side and
    installed into the field's prefetch cache with the scene (hits counted)."""
    import torch
    from paper_2505_00690_b200.envcore import SceneStandby
    from paper_2505_00690_b200.rng import child_seeds_device
    E = 48
    sa, fa, env, ca = _world(E)      # re-samples at each reset
    sb, fb, _, cb = _world(E)        # installs standby scenes
    standby = SceneStandby(sb, env, cb, field=fb if with_field else None)
    rng = np.random.default_rng(5)
    for k in range(25):
        rows = np.flatnonzero(rng.random(E) < 0.12)
        if k % 6 == 1:
            rows = np.union1d(rows, [3])   # a row reset again while its next scene may still be sampling
        if rows.size:
            sl = torch.from_numpy(rows).to("cuda")
            ca[sl] += 1
            cb[sl] += 1
            sa.sample(child_seeds_device(env[sl], "resample", ca[sl]), child_seeds_device(env[sl], "crowd", ca[sl]),
                      slots=sl)
            standby.take(rows)
            fa.set_from_spawn(sa.batch, rows=sl)
            if not with_field:
                fb.set_from_spawn(sb.batch, rows=sl)
        if k % 5 == 0:
            torch.cuda.synchronize()   # let some standby predictions finish before their reset
        fa.step()
        fb.step()
        for name in SCENE:
            assert torch.equal(getattr(sa.batch, name), getattr(sb.batch, name)), (k, name)
        for name in CROWD:
            assert torch.equal(getattr(fa, name), getattr(fb, name)), (k, name)
    sb.batch.check_status()
    if with_field:
        assert fb.stats()["prefetch_hits"] > fa.stats()["prefetch_hits"]


def test_batched_env_standby_equals_resampling(torch_cuda):
    """BatchedEnv(standby=True): resample() installs scenes sampled ahead; trajectories,
    scenes and crowds equal the synchronous re-sampling ones (resets on purpose close
    together, including a slot reset twice in a row)."""
    import torch
    from paper_2505_00690_b200.envcore import BatchedEnv, Scheme
    from paper_2505_00690_b200.urbangen import SceneSpec, TaskKind
    spec = SceneSpec(seed=0, extent_m=(16.0, 16.0), task_kind=TaskKind.NAV_DYNAMIC, pedestrian_count=6)
    K = 12
    envs = [BatchedEnv(spec, Scheme.ASYNC, master_seed=7, k=K, standby=sb) for sb in (False, True)]
    rng = np.random.default_rng(2)
    for t in range(40):
        if t % 4 == 1:
            slots = rng.choice(K, 3, replace=False)
            if t % 8 == 1:
                slots = np.union1d(slots, [4])
            for env in envs:
                env.resample(slots)
        act = rng.uniform(-1, 1, (K, 2))
        for env in envs:
            env.step_batch(act)
        a, b = envs
        assert np.array_equal(np.stack([a.x, a.y, a.vx, a.vy]), np.stack([b.x, b.y, b.vx, b.vy])), t
        assert torch.equal(a.batch.labels, b.batch.labels), t
        assert torch.equal(a.crowd.pos_t, b.crowd.pos_t), t
    assert a.scene_hashes == b.scene_hashes

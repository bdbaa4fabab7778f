"""BASELINE configs at their full per-GPU sizes, through properties that do not
depend on the size (the oracle checks every output bit for bit at smaller env
counts in test_gpu_scale_parity.py):

* cfg3 (4096 envs x 64 peds) and cfg5 (8192 envs x 48 peds): every sampled env is a
  valid scene (labels in {0..3}, every object's centre cell an obstacle, spawn and
  goal cells walkable, starts at least 2 * max radius apart, goal in the start's
  8-connected component, route anchors on walkable cells), rows are independent
  (a re-sample of a few rows leaves the others' bits untouched), and sampling is
  deterministic (a second batch is identical);
* cfg3 dynamics: 20 ticks through CrowdField.run equal 20 synchronous steps for all
  4096 envs, no agent ever inside an obstacle cell."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sample(cfg, E):
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


def _check_scenes(b, res, peds, rows):
    from paper_2505_00690_b200.crowd import connected_components
    labels = b.labels.cpu().numpy()
    assert labels.max() <= 3
    sp_pos, sp_goal = b.sp_pos.cpu().numpy(), b.sp_goal.cpu().numpy()
    kind = b.sp_kind.cpu().numpy()
    routes, nr = b.routes.cpu().numpy(), b.n_routes.cpu().numpy()
    pose, nobj = b.obj_pose.cpu().numpy(), b.obj_n.cpu().numpy()
    rad = np.array([0.3, 0.45, 0.4])
    ny, nx = labels.shape[1:]
    cell = lambda p: (np.floor(p[..., 1] / res).astype(int), np.floor(p[..., 0] / res).astype(int))
    for i in rows:
        lab = labels[i]
        r, c = cell(sp_pos[i, :peds])
        assert (lab[r, c] == 2).all(), i
        gr, gc = cell(sp_goal[i, :peds])
        assert (lab[gr, gc] == 2).all(), i
        d = np.hypot(*(sp_pos[i, :peds, None, :] - sp_pos[i, None, :peds, :]).transpose(2, 0, 1))
        sep = 2.0 * rad[kind[i, :peds]].max()
        assert (d[np.triu_indices(peds, 1)] >= sep - 1e-9).all(), i
        comp = connected_components(lab == 2)
        assert (comp[r, c] == comp[gr, gc]).all(), i
        rr, rc = cell(routes[i, :nr[i]].reshape(-1, 2))
        assert nr[i] >= 1 and (lab[rr, rc] == 2).all(), i
        orr, occ = cell(pose[i, :nobj[i], :2])
        assert (lab[orr, occ] == 0).all(), i   # occupancy.py:49-51


@pytest.mark.parametrize("cfg,E", [("cfg3", 4096), ("cfg5", 8192)])
def test_full_size_sampling_properties(cfg, E, torch_cuda):
    import torch
    s, env = _sample(cfg, E)
    b = s.batch
    b.check_status()
    res = float(b.params.res)
    rng = np.random.default_rng(0)
    rows = rng.choice(E, 48, replace=False)
    _check_scenes(b, res, int(b.params.peds), rows)
    snap = {k: getattr(b, k).clone() for k in ("labels", "elev", "nearest", "sp_pos", "routes", "obj_pose")}
    # row independence: re-sample 5 rows with new seeds, everything else stays bit-identical
    from paper_2505_00690_b200.rng import child_seeds_device
    sl = torch.tensor([3, 100, 1000, E // 2, E - 1], device="cuda")
    new = child_seeds_device(env[sl], "resample", torch.ones(5, dtype=torch.int64, device="cuda"))
    s.sample(new, child_seeds_device(env[sl], "crowd", 1), slots=sl)
    keep = torch.ones(E, dtype=torch.bool, device="cuda")
    keep[sl] = False
    for k, v in snap.items():
        assert torch.equal(getattr(b, k)[keep], v[keep]), k
        assert not torch.equal(getattr(b, k)[sl], v[sl]), k
    # determinism: the original seeds again reproduce the first batch exactly
    s.sample(env[sl], child_seeds_device(env[sl], "crowd", 0), slots=sl)
    for k, v in snap.items():
        assert torch.equal(getattr(b, k), v), k


def test_full_size_cfg3_run_equals_steps(torch_cuda):
    import torch
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
    from paper_2505_00690_b200.rng import child_seeds_device
    s, env = _sample("cfg3", 4096)
    b = s.batch
    seeds = [int(x) for x in child_seeds_device(env, "crowd-run").cpu().numpy().view(np.uint64)]
    f = CrowdField(b, CrowdConfig(), seeds)
    g = CrowdField(b, CrowdConfig(), seeds)
    f.set_from_spawn(b)
    g.set_from_spawn(b)
    labels = b.labels
    nx = labels.shape[2]
    res = float(b.params.res)
    for _ in range(20):
        f.step()
        p = f.pos_t
        r = (p[..., 1] / res).long().clamp(0, nx - 1)
        c = (p[..., 0] / res).long().clamp(0, nx - 1)
        lab = labels.reshape(4096, -1).gather(1, (r * nx + c).reshape(4096, -1))
        assert not bool(((lab == 0) & (f.active_t != 0)).any())
    g.run(20)
    for k in ("pos_t", "vel_t", "goal_t", "waypoint_t", "last_gap_t"):
        assert torch.equal(getattr(f, k), getattr(g, k)), k

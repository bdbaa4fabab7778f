"""cw_crowd_run (CrowdField.run): T ticks without a per-tick barrier across
envs must leave exactly the state of T synchronous CrowdField.step calls --
positions, velocities, goals, waypoints, guidance paths, RNG streams and
last_gap_by_env, bit for bit -- with robots, env masks, split runs, and the
cfg2 shape (256^2 grids, 32 pedestrians, A* replans every tick)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
MIX = {"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}
FIELDS = ("pos_t", "vel_t", "goal_t", "waypoint_t", "path_cells_t", "path_head_t", "path_n_t", "rng_t",
          "last_gap_t", "active_t")


def _pair(E, ext, res, peds, objs, nd=5.0):
    from oracle.rng import child_seed
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec, TaskKind
    seeds = [child_seed(0, "env", i) for i in range(E)]
    area = int(np.floor(4.0 * ext * ext / 100.0 + 0.5))
    spec = SceneSpec(seed=0, extent_m=(ext, ext), task_kind=TaskKind.NAV_DYNAMIC, pedestrian_count=peds,
                     object_density=objs / area, terrain_mix=MIX, grid_resolution_m=res)
    b = SceneSampler(spec, E).sample(seeds, [child_seed(s, "crowd", 0) for s in seeds])
    run = [child_seed(s, "crowd-run") for s in seeds]
    fs = []
    for _ in range(2):
        f = CrowdField(b, CrowdConfig(neighbor_distance=nd), run)
        f.set_from_spawn(b)
        fs.append(f)
    return b, fs


def _robot(b, E, res, seed=3):
    import torch
    g = np.random.default_rng(seed)
    nx = b.params.nx
    walk_n = b.walk_n.cpu().numpy()
    cells = np.array([int(b.walk[e, int(g.integers(walk_n[e]))]) for e in range(E)])
    rp = np.stack([((cells % nx) + 0.5) * res, ((cells // nx) + 0.5) * res], 1)
    rv = g.uniform(-0.5, 0.5, (E, 2))
    return torch.from_numpy(rp).cuda(), torch.from_numpy(rv).cuda()


def _same(a, b, what):
    for k in FIELDS:
        x, y = getattr(a, k).cpu().numpy(), getattr(b, k).cpu().numpy()
        if k == "rng_t":   # Pcg64Raw: state, inc, buffered half, has-half (bytes 40-47 are padding)
            x, y = x[:, :40], y[:, :40]
        assert np.array_equal(x, y), (what, k, np.argwhere(x != y)[:4])


@pytest.mark.parametrize("E,ext,res,peds,objs,T", [(16, 32.0, 0.25, 8, 20, 40),
                                                   (24, 32.0, 0.125, 32, 64, 25),
                                                   (6, 24.0, 0.25, 48, 40, 30)])
def test_run_equals_synchronous_ticks(E, ext, res, peds, objs, T, torch_cuda):
    b, (f, g) = _pair(E, ext, res, peds, objs)
    rp, rv = _robot(b, E, res)
    for _ in range(T):
        f.step(rp, rv, 0.35)
    g.run(T, rp, rv, 0.35)
    torch_cuda.cuda.synchronize()
    _same(f, g, "run")
    assert np.isfinite(g.last_gap_t.cpu().numpy()).any()


def test_run_with_env_mask_and_split_runs(torch_cuda):
    import torch
    E, T = 12, 30
    b, (f, g) = _pair(E, 32.0, 0.25, 8, 20)
    rp, rv = _robot(b, E, 0.25, seed=9)
    mask = torch.from_numpy((np.arange(E) % 3 != 1).astype(np.uint8)).cuda()
    for _ in range(T):
        f.step(rp, rv, 0.35, env_mask=mask)
    g.run(11, rp, rv, 0.35, env_mask=mask)
    g.run(1, rp, rv, 0.35, env_mask=mask)
    g.run(T - 12, rp, rv, 0.35, env_mask=mask)
    _same(f, g, "masked split run")


def test_run_in_chunks_matches(torch_cuda):
    """A run longer than one call's history budget goes in chunks; same state."""
    E = 8
    b, (f, g) = _pair(E, 32.0, 0.25, 8, 20)
    g.run_history_bytes = 8 * E * 7      # 7 ticks per call
    for _ in range(23):
        f.step()
    g.run(23)
    _same(f, g, "chunked")


def test_run_without_robot_then_steps(torch_cuda):
    E = 8
    b, (f, g) = _pair(E, 32.0, 0.25, 8, 20)
    for _ in range(15):
        f.step()
    g.run(15)
    _same(f, g, "no robot")
    for _ in range(3):   # synchronous ticks continue from the run's state
        f.step()
        g.step()
    _same(f, g, "after run")


def test_run_edge_cases(torch_cuda):
    """One env, one tick, one agent; every env masked; an open arena (no obstacles,
    so no searches at all); run(0) is a no-op."""
    import torch
    from paper_2505_00690_b200.crowd import CrowdAgent, CrowdConfig, CrowdField
    from paper_2505_00690_b200.urbangen import OccupancyGrid
    b, (f, g) = _pair(1, 16.0, 0.25, 1, 4)
    for _ in range(1):
        f.step()
    g.run(1)
    _same(f, g, "E=1 T=1")
    g.run(0)
    _same(f, g, "run(0)")
    b, (f, g) = _pair(6, 32.0, 0.25, 8, 20)
    mask = torch.zeros(6, dtype=torch.uint8, device="cuda")
    for _ in range(5):
        f.step(env_mask=mask)
    g.run(5, env_mask=mask)
    _same(f, g, "all masked")
    ny = nx = 64
    occ = OccupancyGrid(0.25, np.full((ny, nx), 2, np.uint8), np.zeros((ny, nx), np.float32))
    rng = np.random.default_rng(5)
    agents = [[CrowdAgent(i, rng.uniform(1, 15, 2), np.zeros(2), 0.3, 1.2, rng.uniform(1, 15, 2))
               for i in range(12)] for _ in range(3)]
    fs = []
    for _ in range(2):
        h = CrowdField([occ] * 3, CrowdConfig(), [11, 12, 13])
        h.set_agents(agents)
        fs.append(h)
    for _ in range(40):
        fs[0].step()
    fs[1].run(40)
    _same(fs[0], fs[1], "open arena")


def test_run_full_cfg2_batch_matches_steps(torch_cuda):
    """1024 cfg2 envs x 30 ticks: every env's state equals 30 synchronous steps."""
    b, (f, g) = _pair(1024, 32.0, 0.125, 32, 64)
    rp, rv = _robot(b, 1024, 0.125, seed=21)
    for _ in range(30):
        f.step(rp, rv, 0.35)
    g.run(30, rp, rv, 0.35)
    _same(f, g, "cfg2 x 1024")


def test_run_long_horizon_matches_steps(torch_cuda):
    """256 cfg2 envs x 400 ticks in one run call (goals re-drawn many times, RNG
    streams advanced far): bit-identical to 400 synchronous steps, and the
    bench's per-env state checksum agrees."""
    from paper_2505_00690_b200 import shard
    b, (f, g) = _pair(256, 32.0, 0.125, 32, 64)
    rp, rv = _robot(b, 256, 0.125, seed=5)
    for _ in range(400):
        f.step(rp, rv, 0.35, check=False)
    f.check_flags()
    g.run(400, rp, rv, 0.35)
    _same(f, g, "cfg2 x 256 x 400 ticks")
    assert np.array_equal(shard.state_checksum(f.pos_t, f.vel_t, f.goal_t, f.last_gap_t).cpu().numpy(),
                          shard.state_checksum(g.pos_t, g.vel_t, g.goal_t, g.last_gap_t).cpu().numpy())


def test_run_binned_warp_path(torch_cuda):
    """A >= 128 (cell-binned neighbour search, warp-per-agent rounds) on a block layout."""
    from oracle.rng import child_seed
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec, TaskKind
    seeds = [child_seed(0, "env", 40 + i) for i in range(3)]
    spec = SceneSpec(seed=0, extent_m=(48.0, 48.0), task_kind=TaskKind.NAV_CLEAR, object_density=0.0,
                     pedestrian_count=140, terrain_mix=MIX, grid_resolution_m=0.25)
    b = SceneSampler(spec, 3).sample(seeds, [child_seed(s, "crowd", 0) for s in seeds])
    run = [child_seed(s, "crowd-run") for s in seeds]
    fs = []
    for _ in range(2):
        f = CrowdField(b, CrowdConfig(neighbor_distance=3.0), run)
        f.set_from_spawn(b)
        fs.append(f)
    rp, rv = _robot(b, 3, 0.25, seed=4)
    for _ in range(12):
        fs[0].step(rp, rv, 0.35)
    fs[1].run(12, rp, rv, 0.35)
    _same(fs[0], fs[1], "A=140 binned")


@pytest.mark.parametrize("overlap", [False, True])
def test_run_with_resampling_matches_synchronous_driver(overlap, torch_cuda):
    """cfg5-style driver: ~10 % of envs re-sampled before each tick.  The segmented
    run (envcore.run_with_resampling: cw_crowd_run_window between batched
    re-samples) leaves the state of re-sampling + stepping tick by tick."""
    import torch
    from oracle.rng import child_seed
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
    from paper_2505_00690_b200.envcore import run_with_resampling
    from paper_2505_00690_b200.rng import child_seeds_device, seeds_to_tensor
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec, TaskKind
    E, T = 16, 40
    seeds = [child_seed(0, "env", i) for i in range(E)]
    spec = SceneSpec(seed=0, extent_m=(32.0, 32.0), task_kind=TaskKind.NAV_DYNAMIC, pedestrian_count=8,
                     object_density=20 / 41, terrain_mix=MIX, grid_resolution_m=0.25)
    rng = np.random.default_rng(8)
    events = [np.flatnonzero(rng.random(E) < 0.1) for _ in range(T)]
    out = []
    for mode in ("sync", "run"):
        sampler = SceneSampler(spec, E)
        b = sampler.sample(seeds, [child_seed(s, "crowd", 0) for s in seeds])
        f = CrowdField(b, CrowdConfig(), [child_seed(s, "crowd-run") for s in seeds])
        f.set_from_spawn(b)
        env_t = seeds_to_tensor(seeds, "cuda")
        counts = torch.zeros(E, dtype=torch.int64, device="cuda")
        rp, rv = _robot(b, E, 0.25, seed=2)
        if mode == "sync":
            for t in range(T):
                if len(events[t]):
                    sl = torch.as_tensor(events[t], dtype=torch.int64, device="cuda")
                    counts[sl] += 1
                    sampler.sample(child_seeds_device(env_t[sl], "resample", counts[sl]),
                                   child_seeds_device(env_t[sl], "crowd", counts[sl]), slots=sl)
                    f.set_from_spawn(b, rows=sl)
                f.step(rp, rv, 0.35)
        else:
            n = run_with_resampling(sampler, f, env_t, counts, events, T, rp, rv, 0.35, overlap=overlap)
            assert n == sum(len(x) for x in events)
        torch_cuda.cuda.synchronize()
        out.append((f, b.labels.cpu().numpy()))
    assert np.array_equal(out[0][1], out[1][1])
    _same(out[0][0], out[1][0], "resampling driver")


@pytest.mark.parametrize("case", range(6))
def test_run_random_configs(case, torch_cuda):
    """Seeded random shapes (agent counts 1..130 across the lane / binned paths, grid sizes,
    resolutions, densities, neighbour radii, robots on / off, random env masks): a run
    equals the same number of synchronous steps."""
    import torch
    from oracle.rng import child_seed
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec, TaskKind
    r = np.random.default_rng(100 + case)
    A = int([1, 5, 17, 40, 70, 130][case])
    E = int(r.integers(2, 12))
    res = float(r.choice([0.1, 0.2, 0.25]))
    ext = float(r.choice([12.0, 20.0, 32.0])) if A < 100 else 48.0
    task = TaskKind.NAV_DYNAMIC if A < 100 else TaskKind.NAV_CLEAR
    nd = float(r.choice([3.0, 5.0]))
    T = int(r.integers(10, 40))
    seeds = [child_seed(0, "env", 1000 * case + i) for i in range(E)]
    spec = SceneSpec(seed=0, extent_m=(ext, ext), task_kind=task, pedestrian_count=A,
                     object_density=float(r.uniform(0.2, 1.5)) if task == TaskKind.NAV_DYNAMIC else 0.0,
                     terrain_mix=MIX, grid_resolution_m=res)
    b = SceneSampler(spec, E).sample(seeds, [child_seed(s, "crowd", 0) for s in seeds])
    run = [child_seed(s, "crowd-run") for s in seeds]
    fs = []
    for _ in range(2):
        f = CrowdField(b, CrowdConfig(neighbor_distance=nd), run)
        f.set_from_spawn(b)
        fs.append(f)
    robot = case % 2 == 0
    rp, rv = _robot(b, E, res, seed=case) if robot else (None, None)
    mask = torch.from_numpy((r.random(E) < 0.8).astype(np.uint8)).cuda() if case % 3 == 1 else None
    for _ in range(T):
        fs[0].step(rp, rv, 0.35, env_mask=mask)
    fs[1].run(T, rp, rv, 0.35, env_mask=mask)
    _same(fs[0], fs[1], f"random case {case}: E={E} A={A} ext={ext} res={res} nd={nd} T={T}")


def test_run_as_first_crowd_launch_of_a_process(tmp_path):
    """A run whose kernels are the process's first crowd launches (no prior step):
    the run reserves its kernels' local memory before starting the persistent
    server, so no launch can wait on a driver resize while the server runs."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import numpy as np, torch\n"
        "from test_gpu_run import _pair\n"
        "b, (f, g) = _pair(8, 32.0, 0.125, 32, 64)\n"
        "f.run(6)\n"
        "for _ in range(6): g.step()\n"
        "assert np.array_equal(f.pos_t.cpu().numpy(), g.pos_t.cpu().numpy())\n"
        "print('ok')\n" % (root, os.path.join(root, "tests")))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]

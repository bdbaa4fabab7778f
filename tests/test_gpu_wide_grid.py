"""Crowd on grids wider or taller than 1024 cells (the reference's Traverse strip preset,
bench/presets.py:50-60: 120 m x 10 m at the default 0.1 m = 1200 x 100 cells, and its
transpose), through the C ABI, bit-exact against the oracle.  The A* keys pack the cell as
row << cb | col with cb = ceil(log2 nx) there (astar.cuh make_key2), so these grids
exercise the non-default packing; 60 ticks with a robot in the lane make every agent
replan through obstacles."""

import numpy as np
import pytest

from conftest import golden_catalog

pytestmark = pytest.mark.gpu

MIX = {"Flat": 0.4, "Slope": 0.2, "Stair": 0.2, "Rough": 0.2}   # presets.py:17


@pytest.mark.parametrize("ext,task", [((120.0, 10.0), "Traverse"), ((10.0, 120.0), "NavStatic"),
                                      ((150.0, 6.0), "NavDynamic")])
def test_wide_grid_crowd_matches_oracle(ext, task, torch_cuda):
    from oracle import crowd as C
    from oracle import scene as S
    from oracle.rng import child_seed
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField, spawn_agents
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec, TaskKind
    res, peds, E = 0.1, 8, 2
    seeds = [child_seed(3, "env", i) for i in range(E)]
    spec = SceneSpec(seed=seeds[0], extent_m=ext, task_kind=TaskKind(task), object_density=1.0,
                     pedestrian_count=peds, terrain_mix=MIX, grid_resolution_m=res)
    b = SceneSampler(spec, E).sample(seeds, [child_seed(s, "crowd", 0) for s in seeds])
    grids, dev_agents, ref_agents = [], [], []
    for i, s in enumerate(seeds):
        sc = S.generate_scene(dict(seed=s, extent=ext, res=res, task=task, split="Train",
                                   density=1.0, mix=MIX), golden_catalog())
        assert np.array_equal(b.labels[i].cpu().numpy(), sc["labels"]), i
        ny, nx = sc["labels"].shape
        assert max(nx, ny) > 1024
        grids.append((sc["labels"], res))
        sp = C.spawn_agents(sc["labels"], res, peds, child_seed(s, "crowd", 0))
        ag = spawn_agents(b.occupancy(i), peds, child_seed(s, "crowd", 0))
        assert np.array_equal(np.array([a.position for a in ag]), sp["pos"]), i
        dev_agents.append(ag)
        ref_agents.append(sp)
    run = [child_seed(s, "crowd-run") for s in seeds]
    f = CrowdField(b, CrowdConfig(), run)
    f.set_agents(dev_agents)
    ref = C.CrowdFieldOracle(grids, C.Config(), run)
    ref.set_agents(ref_agents)
    # the robot crosses the middle of the strip
    rp = np.array([[ext[0] * 0.5, ext[1] * 0.5]] * E)
    rv = np.array([[0.6, 0.0] if ext[0] > ext[1] else [0.0, 0.6]] * E)
    for t in range(60):
        f.step(robot_pos=rp, robot_vel=rv)
        ref.step(robot_pos=rp, robot_vel=rv)
        assert np.array_equal(f.pos, ref.pos), t
        assert np.array_equal(f.vel, ref.vel), t
        rp = rp + rv * 0.05
    assert np.array_equal(f.goal, ref.goal)
    assert f.stats()["astar_expansions"] > 0   # the searches ran on the wide packing


def test_wide_grid_run_equals_steps(torch_cuda):
    """CrowdField.run on a 1200 x 100 strip (stepped tick by tick there) equals steps."""
    from oracle.rng import child_seed
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec, TaskKind
    seeds = [child_seed(5, "env", i) for i in range(2)]
    spec = SceneSpec(seed=seeds[0], extent_m=(120.0, 10.0), task_kind=TaskKind.NAV_DYNAMIC,
                     object_density=1.0, pedestrian_count=12, terrain_mix=MIX, grid_resolution_m=0.1)
    b = SceneSampler(spec, 2).sample(seeds, [child_seed(s, "crowd", 0) for s in seeds])
    run = [child_seed(s, "crowd-run") for s in seeds]
    fa, fb = CrowdField(b, CrowdConfig(), run), CrowdField(b, CrowdConfig(), run)
    fa.set_from_spawn(b)
    fb.set_from_spawn(b)
    rp, rv = np.array([[60.0, 5.0]] * 2), np.zeros((2, 2))
    fa.run(30, robot_pos=rp, robot_vel=rv)
    for _ in range(30):
        fb.step(robot_pos=rp, robot_vel=rv)
    assert np.array_equal(fa.pos, fb.pos) and np.array_equal(fa.vel, fb.vel)

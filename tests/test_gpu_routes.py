"""Device route anchors + robot spawn vs fixtures from the unmodified reference
(tests/golden/routes.npz, oracle/make_golden_routes.py): bit-exact routes for 21
scenes (courtyard 128^2 / 256^2, block layouts 192^2, small NavStatic, Traverse
strips) and the spawn poses BatchedEnv draws from them."""

import json

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu
MIX = {"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}


def _spec(d):
    from paper_2505_00690_b200.urbangen import SceneSpec, TaskKind
    return SceneSpec(seed=int(d["seed"]), extent_m=(d["extent"], d["extent"]), task_kind=TaskKind(d["task"]),
                     object_density=d["density"], pedestrian_count=0, terrain_mix=MIX,
                     grid_resolution_m=d["res"])


@pytest.mark.parametrize("case", range(21))
def test_route_anchors_match_reference(case, torch_cuda):
    from paper_2505_00690_b200.urbangen import SceneSampler
    g = load_golden("routes.npz")
    d = json.loads(str(g[f"c{case}_spec"]))
    b = SceneSampler(_spec(d), 1).sample([int(d["seed"])])
    assert np.array_equal(b.labels[0].cpu().numpy(), g[f"c{case}_labels"])
    n = int(b.n_routes[0])
    want = g[f"c{case}_routes"]
    assert n == want.shape[0]
    assert np.array_equal(b.routes[0, :n].cpu().numpy(), want)


@pytest.mark.parametrize("case", [0, 5, 12])
def test_batched_env_spawns_on_reference_route(case, torch_cuda):
    from paper_2505_00690_b200.envcore import BatchedEnv, Scheme
    g = load_golden("routes.npz")
    d = json.loads(str(g[f"c{case}_spec"]))
    env = BatchedEnv(_spec(d), Scheme.ASYNC, master_seed=0, k=1, env_seeds=[int(d["seed"])])
    (sx, sy), (gx, gy) = g[f"c{case}_routes"][int(g[f"c{case}_spawn_pick"][0])]
    st = env.robot_state(0)
    assert (st["x"], st["y"]) == (sx, sy) and st["goal"] == [gx, gy]
    assert st["yaw"] == float(np.arctan2(gy - sy, gx - sx))

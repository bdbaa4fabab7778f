"""Process-pool workers for the at-scale parity sweep (tests/test_gpu_scale_parity.py).

Test infrastructure only (the checker, never the product): each worker restates
one env of a BASELINE config with the oracle -- the scene as BatchedEnv samples
it (urbangen/scene.py:38-88 generate_scene incl. raster, scene.py:102-158 route
anchors, crowd/step.py:37 spawn_agents, field.py:571 nearest-obstacle map) or
T crowd ticks of that env (field.py:90-163) with the bench's static robot.
"""

import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MIX = {"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}


def _catalog():
    from . import scene as S
    path = os.path.join(HERE, "..", "paper_2505_00690_b200", "data", "catalog.json")
    return S.load_catalog_tuples(json.load(open(path)))


def density(extent, res, objects):
    n = int(np.ceil(extent / res))
    base = int(np.floor(4.0 * (n * n * res * res) / 100.0 + 0.5))
    return objects / base if objects else 0.0


def sample_env(job):
    """job = (env_id, extent, res, objects, peds, task) -> dict of the env's sample."""
    from . import crowd as C
    from . import routes as R
    from . import scene as S
    from .rng import child_seed
    env_id, extent, res, objects, peds, task = job
    s = child_seed(0, "env", env_id)
    sc = S.generate_scene(dict(seed=s, extent=(extent, extent), res=res, task=task, split="Train",
                               density=density(extent, res, objects), mix=MIX), _catalog())
    out = {"zones": sc["zones"], "assign": sc["assign"], "labels": sc["labels"],
           "elev_bits": sc["elev"].view(np.uint32), "overflow": bool(sc["overflow"]),
           "objects": np.array([[k, x, y, yaw] for k, x, y, yaw in sc["objects"]], np.float64).reshape(-1, 4)}
    near = C.nearest_obstacle_map(sc["labels"])
    out["nearest"] = None if near is None else near.astype(np.int32)
    out["walk_n"] = int((sc["labels"] == 2).sum())
    if peds:
        sp = C.spawn_agents(sc["labels"], res, peds, child_seed(s, "crowd", 0))
        out.update(sp_pos=np.asarray(sp["pos"]), sp_goal=np.asarray(sp["goal"]), sp_kind=sp["kind"],
                   sp_pref=sp["pref"])
    rt = R.sample_route_anchors(sc["labels"], res, s, (extent, extent), task)
    out["routes"] = None if rt is None else np.array(rt, np.float64).reshape(-1, 2, 2)
    return out


def step_env(job):
    """job = (env_id, extent, res, objects, peds, task, nd, ticks, robot_u) -> final
    pos, vel, goal, waypoint, last gap after ``ticks`` ticks from spawn."""
    from . import crowd as C
    from . import scene as S
    from .rng import child_seed
    env_id, extent, res, objects, peds, task, nd, ticks, robot_u = job
    s = child_seed(0, "env", env_id)
    sc = S.generate_scene(dict(seed=s, extent=(extent, extent), res=res, task=task, split="Train",
                               density=density(extent, res, objects), mix=MIX), _catalog())
    labels = sc["labels"]
    sp = C.spawn_agents(labels, res, peds, child_seed(s, "crowd", 0))
    f = C.CrowdFieldOracle([(labels, res)], C.Config(neighbor_distance=nd), [child_seed(s, "crowd-run")])
    f.set_agents([sp])
    walk = np.flatnonzero(labels.reshape(-1) == 2)
    c = int(walk[int(robot_u * len(walk))])
    nx = labels.shape[1]
    rp = np.array([[(c % nx + 0.5) * res, (c // nx + 0.5) * res]])
    rv = np.zeros((1, 2))
    gaps = []
    for _ in range(ticks):
        f.step(robot_pos=rp, robot_vel=rv, robot_radius=0.35)
        gaps.append(float(f.last_gap_by_env[0]))
    return {"pos": f.pos[0].copy(), "vel": f.vel[0].copy(), "goal": f.goal[0].copy(),
            "waypoint": f.waypoint[0].copy(), "gaps": np.array(gaps), "robot": rp[0]}

"""Generate tests/golden/robot_*.npz from the REAL reference (build container only).

Run:  PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_robot.py
Drives the unmodified reference's BatchedEnv.step_batch (envcore/batch.py:205-302:
crowd step with the robot lane, integrate_motion, traversability gating, crowd
contact, reward_batch, observe_batch) with seeded random actions and stores every
tick's robot state, events, rewards and observations, plus each env's
traversability_maps (robot.py:127-179).  Read by tests/test_robot_golden.py (oracle
pinning, CPU) and tests/test_gpu_robot.py (device parity).
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
MIX = {"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}

# (name, robot, K, T, peds, extent, res, density, horizon, auto_reset)
RUNS = [
    ("quadruped", "quadruped", 4, 120, 8, 32.0, 0.25, 20 / 41, 200, False),
    ("wheeled", "wheeled", 2, 40, 4, 32.0, 0.25, 20 / 41, 25, True),
    ("small", "humanoid", 6, 90, 3, 12.0, 0.2, 0.5, 60, False),
]


def main():
    sys.path.insert(0, REF)
    from citywalk.envcore.batch import BatchedEnv, EnvConfig, Scheme
    from citywalk.envcore.robot import ROBOT_MODELS, traversability_maps
    from citywalk.rng import child_seed
    from citywalk.urbangen import SceneSpec, TaskKind

    os.makedirs(OUT, exist_ok=True)
    for name, robot, K, T, peds, ext, res, dens, horizon, auto in RUNS:
        spec = SceneSpec(seed=0, extent_m=(ext, ext), task_kind=TaskKind.NAV_DYNAMIC,
                         object_density=dens, pedestrian_count=peds, terrain_mix=MIX,
                         grid_resolution_m=res)
        cfg = EnvConfig(robot=robot, horizon=horizon, auto_reset=auto)
        env = BatchedEnv(spec, Scheme.ASYNC, master_seed=0, k=K, config=cfg)
        model = ROBOT_MODELS[robot]
        maps = [traversability_maps(env.occs[i], model) for i in range(K)]
        out = dict(
            env_seeds=np.array(env.env_seeds, np.uint64),
            passable=np.stack([m["passable"] for m in maps]).astype(np.uint8),
            obstacle=np.stack([m["obstacle"] for m in maps]).astype(np.uint8),
            step=np.stack([m["step"] for m in maps]), grade=np.stack([m["grade"] for m in maps]),
            rough=np.stack([m["rough"] for m in maps]),
            labels=env.labels_stack.copy(), grid_elev=env.elev_stack.copy(),
        )
        rng = np.random.default_rng(77)
        keys = ("x", "y", "yaw", "vx", "vy", "elev", "tick", "terminated", "truncated")
        rec = {k: [] for k in keys}
        rec0 = {k: np.array(getattr(env, k)).copy() for k in keys}
        rec0["goal"] = env.goal.copy()
        acts, rew, ev, depth, gvec, pvel, hmap, cpos, cvel, goals = [], [], [], [], [], [], [], [], [], []
        evk = ("collision", "collision_static", "collision_dynamic", "on_walkable", "reached",
               "out_of_bounds")
        dist, pinc = [], []
        for t in range(T):
            # mostly forward (collisions, walls, out-of-bounds), some out-of-range values (clipped)
            a = np.stack([rng.uniform(0.2, 1.3, K), rng.uniform(-0.7, 0.7, K)], axis=-1)
            res_t = env.step_batch(a)
            acts.append(a)
            for k in keys:
                rec[k].append(np.array(getattr(env, k)).copy())
            goals.append(env.goal.copy())
            rew.append([r.reward for r in res_t])
            ev.append([[r.events[k] for k in evk] for r in res_t])
            dist.append([r.events["distance_to_goal"] for r in res_t])
            pinc.append([r.events["path_increment"] for r in res_t])
            depth.append(np.stack([r.observation.depth for r in res_t]))
            gvec.append(np.stack([r.observation.goal_vector for r in res_t]))
            pvel.append([r.observation.projected_velocity for r in res_t])
            hmap.append(np.stack([r.observation.height_map for r in res_t]))
            cpos.append(env.crowd.pos.copy())
            cvel.append(env.crowd.vel.copy())
        out.update({f"init_{k}": v for k, v in rec0.items()})
        out.update({k: np.array(v) for k, v in rec.items()})
        out.update(actions=np.array(acts), reward=np.array(rew), events=np.array(ev, bool),
                   distance=np.array(dist), path_inc=np.array(pinc), depth=np.array(depth),
                   goal_vector=np.array(gvec), proj_vel=np.array(pvel), height_map=np.array(hmap),
                   crowd_pos=np.array(cpos), crowd_vel=np.array(cvel), goal=np.array(goals),
                   crowd_radius=env.crowd.radius.copy(), crowd_active=env.crowd.active.copy(),
                   meta=np.array([K, T, peds, horizon, int(auto)], np.int64),
                   res=np.float64(res), extent=np.float64(ext), density=np.float64(dens),
                   robot=np.array(robot))
        np.savez_compressed(os.path.join(OUT, f"robot_{name}.npz"), **out)
        print(name, "written")


if __name__ == "__main__":
    main()

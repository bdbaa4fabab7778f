"""Drift of BatchedEnv.step_batch (device) from the reference golden over 120 ticks (GPU)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_golden
from paper_2505_00690_b200.envcore import BatchedEnv, EnvConfig, Scheme
from paper_2505_00690_b200.urbangen import SceneSpec, TaskKind
g = load_golden("robot_quadruped.npz")
K, T = int(g["meta"][0]), int(g["meta"][1])
spec = SceneSpec(seed=0, extent_m=(32.0, 32.0), task_kind=TaskKind.NAV_DYNAMIC, object_density=20 / 41, pedestrian_count=8,
                 terrain_mix={"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}, grid_resolution_m=0.25)
env = BatchedEnv(spec, Scheme.ASYNC, master_seed=0, k=K, config=EnvConfig(robot="quadruped"))
env.set_robot_state(g["init_x"], g["init_y"], g["init_yaw"], g["init_goal"], elev=g["init_elev"])
for t in range(T):
    res = env.step_batch(g["actions"][t])
    cp = np.abs(env.crowd.pos - g["crowd_pos"][t]).max(); cv = np.abs(env.crowd.vel - g["crowd_vel"][t]).max()
    rx = max(abs(env.robot_state(i)["x"] - g["x"][t][i]) for i in range(K))
    if t % 10 == 9 or cp > 0:
        print(t, f"crowd pos {cp:.2e} vel {cv:.2e} robot x {rx:.2e}")

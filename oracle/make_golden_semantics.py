"""Generate tests/golden/robot_semantics.npz from the REAL reference (build container only).

Run:  PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_semantics.py
Calls the unmodified reference's observe_batch(include_semantics=True)
(envcore/observe.py:39-129; the per-ray label of the hit cell at observe.py:84-85,
0 for rays that reach the cap or leave the grid) on every post-step robot state of
the robot goldens (tests/golden/robot_{quadruped,small}.npz, themselves written by
oracle/make_golden_robot.py from BatchedEnv.step_batch), and stores the
semantics and depth per tick.  In those scenes every ray stops at an OBSTACLE
(label 0) or at the cap, so a synthetic case adds the rise walls: seeded 64 x 48
grids of random labels (few obstacles) over a terraced elevation field (steps of
0.02-0.4 m, wheeled max_step_rise 0.05 m), 16 robots at seeded poses.  Read by tests/test_robot_golden.py (oracle
pinning, CPU) and tests/test_gpu_robot.py (device parity).
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
RUNS = ("quadruped", "small")


def main():
    sys.path.insert(0, REF)
    from citywalk.envcore.observe import observe_batch
    from citywalk.envcore.robot import ROBOT_MODELS

    out = {}
    for name in RUNS:
        g = np.load(os.path.join(GOLD, f"robot_{name}.npz"))
        rise = ROBOT_MODELS[str(g["robot"])].max_step_rise
        T = g["x"].shape[0]
        sem, depth = [], []
        for t in range(T):
            vel = np.stack([g["vx"][t], g["vy"][t]], -1)
            o = observe_batch(g["x"][t], g["y"][t], g["yaw"][t], g["goal"][t], vel, g["elev"][t],
                              g["labels"], g["grid_elev"], float(g["res"]), rise, include_semantics=True)
            sem.append(o["semantics"])
            depth.append(o["depth"])
        out[f"{name}_semantics"] = np.array(sem, np.uint8)
        out[f"{name}_depth"] = np.array(depth, np.float32)
        u, c = np.unique(out[f"{name}_semantics"], return_counts=True)
        print(name, T, dict(zip(u.tolist(), c.tolist())))
    # synthetic terraces: rays stop on rises over walkable / roadway / ground cells
    rng = np.random.default_rng(2505)
    K, ny, nx, res = 16, 48, 64, 0.25
    labels = rng.choice(np.array([0, 1, 2, 3], np.uint8), size=(K, ny, nx), p=[0.02, 0.2, 0.5, 0.28])
    steps = rng.uniform(0.02, 0.4, size=(K, ny // 4, nx // 4)).astype(np.float32)
    elev = np.cumsum(np.kron(steps, np.ones((4, 4), np.float32)) * (rng.random((K, ny, nx)) < 0.15),
                     axis=2).astype(np.float32)
    x = rng.uniform(0.5, nx * res - 0.5, K)
    y = rng.uniform(0.5, ny * res - 0.5, K)
    yaw = rng.uniform(-np.pi, np.pi, K)
    goal = np.stack([rng.uniform(0, nx * res, K), rng.uniform(0, ny * res, K)], -1)
    vel = rng.normal(size=(K, 2))
    r, c = (y / res).astype(np.int64), (x / res).astype(np.int64)
    er = elev[np.arange(K), r, c].astype(np.float64)
    o = observe_batch(x, y, yaw, goal, vel, er, labels, elev, res, 0.05, include_semantics=True)
    out.update(synth_labels=labels, synth_elev=elev, synth_x=x, synth_y=y, synth_yaw=yaw, synth_goal=goal,
               synth_vel=vel, synth_er=er, synth_res=np.float64(res), synth_rise=np.float64(0.05),
               synth_semantics=o["semantics"].astype(np.uint8), synth_depth=o["depth"],
               synth_goal_vector=o["goal_vector"], synth_proj_vel=o["projected_velocity"],
               synth_height_map=o["height_map"])
    u, c = np.unique(o["semantics"], return_counts=True)
    print("synth", dict(zip(u.tolist(), c.tolist())), "hits", int((o["depth"] < 10).sum()))
    np.savez_compressed(os.path.join(GOLD, "robot_semantics.npz"), **out)


if __name__ == "__main__":
    main()

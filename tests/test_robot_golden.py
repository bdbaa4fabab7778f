"""Pin oracle/robot.py (traversability, robot step, reward, observations) to
fixtures generated from the unmodified reference (oracle/make_golden_robot.py)."""

import numpy as np
import pytest

from conftest import load_golden

RUNS = ["quadruped", "wheeled", "small"]


def _steps_before_reset(g):
    tick = g["tick"][:, 0]
    drop = np.flatnonzero(np.diff(tick) < 0)
    return int(drop[0]) + 1 if drop.size else tick.shape[0]


@pytest.mark.parametrize("run", RUNS)
def test_traversability_maps_match_reference(run):
    from oracle import robot as R
    g = load_golden(f"robot_{run}.npz")
    m = R.MODELS[str(g["robot"])]
    for i in range(g["labels"].shape[0]):
        q = R.traversability_maps(g["labels"][i], g["grid_elev"][i], float(g["res"]), m)
        for k in ("passable", "obstacle"):
            assert np.array_equal(q[k].astype(np.uint8), g[k][i]), (i, k)
        for k in ("step", "grade", "rough"):
            assert np.array_equal(q[k], g[k][i]), (i, k)


@pytest.mark.parametrize("run", RUNS)
def test_robot_step_replays_reference(run):
    from oracle import robot as R
    g = load_golden(f"robot_{run}.npz")
    K, T, peds, horizon, auto = (int(v) for v in g["meta"])
    rb = R.RobotBatch(g["labels"], g["grid_elev"], float(g["res"]), str(g["robot"]), horizon=horizon)
    for k in ("x", "y", "yaw", "vx", "vy"):
        setattr(rb, k, g[f"init_{k}"].copy())
    rb.el = g["init_elev"].copy()
    rb.goal = g["init_goal"].copy()
    names = ("collision", "collision_static", "collision_dynamic", "on_walkable", "reached",
             "out_of_bounds")
    n = _steps_before_reset(g) if auto else T
    for t in range(n):
        rew, ev, obs = rb.step(g["actions"][t], g["crowd_pos"][t], g["crowd_radius"], g["crowd_active"])
        for k, a in (("x", rb.x), ("y", rb.y), ("yaw", rb.yaw), ("vx", rb.vx), ("vy", rb.vy),
                     ("elev", rb.el), ("tick", rb.tick), ("terminated", rb.terminated),
                     ("truncated", rb.truncated)):
            assert np.array_equal(a, g[k][t]), (t, k)
        assert np.array_equal(rew, g["reward"][t]), t
        for j, k in enumerate(names):
            assert np.array_equal(ev[k], g["events"][t, :, j]), (t, k)
        assert np.array_equal(ev["distance"], g["distance"][t]), t
        assert np.array_equal(ev["path_inc"], g["path_inc"][t]), t
        for k in ("depth", "goal_vector", "proj_vel", "height_map"):
            assert np.array_equal(obs[k], g[k][t]), (t, k)
    assert n > 20


def test_reach_and_out_of_bounds_terminate():
    """Terminal rewards fire on the reach / out-of-bounds step (reward.py:29-53,
    batch.py:272-281) -- constructed states, oracle only."""
    from oracle import robot as R
    n = 40
    labels = np.full((2, n, n), 2, np.uint8)
    elev = np.zeros((2, n, n), np.float32)
    rb = R.RobotBatch(labels, elev, 0.25, "quadruped", horizon=5)
    rb.x[:] = [5.0, 9.9]
    rb.y[:] = [5.0, 5.0]
    rb.goal[:] = [[5.05, 5.0], [1.0, 1.0]]
    rew, ev, _ = rb.step(np.array([[1.0, 0.0], [1.0, 0.0]]))
    assert ev["reached"][0] and not ev["reached"][1]
    assert ev["out_of_bounds"][1] and not ev["out_of_bounds"][0]
    assert rew[0] > 50.0 and rew[1] < -90.0
    assert rb.terminated.all()
    rew2, _, _ = rb.step(np.zeros((2, 2)))
    assert (rew2 == 0.0).all() and (rb.tick == 1).all()


@pytest.mark.parametrize("run", ["quadruped", "small"])
def test_observe_semantics_match_reference(run):
    """observe.py:84-85 per-ray semantics on every post-step state of the robot goldens
    (oracle/make_golden_semantics.py)."""
    from oracle import robot as R
    g = load_golden(f"robot_{run}.npz")
    s = load_golden("robot_semantics.npz")
    rise = R.MODELS[str(g["robot"])].max_step_rise
    for t in range(g["x"].shape[0]):
        vel = np.stack([g["vx"][t], g["vy"][t]], -1)
        o = R.observe(g["x"][t], g["y"][t], g["yaw"][t], g["goal"][t], vel, g["elev"][t],
                      g["labels"], g["grid_elev"], float(g["res"]), rise)
        assert np.array_equal(o["semantics"], s[f"{run}_semantics"][t]), t
        assert np.array_equal(o["depth"], s[f"{run}_depth"][t]), t


def test_observe_semantics_rise_walls_match_reference():
    """Synthetic terraces: rays stopped by rises carry the walkable / roadway / ground
    label of the cell they stop in (labels 1-3 present in the fixture)."""
    from oracle import robot as R
    s = load_golden("robot_semantics.npz")
    o = R.observe(s["synth_x"], s["synth_y"], s["synth_yaw"], s["synth_goal"], s["synth_vel"],
                  s["synth_er"], s["synth_labels"], s["synth_elev"], float(s["synth_res"]),
                  float(s["synth_rise"]))
    assert set(np.unique(s["synth_semantics"]).tolist()) == {0, 1, 2, 3}
    assert np.array_equal(o["semantics"], s["synth_semantics"])
    assert np.array_equal(o["depth"], s["synth_depth"])
    assert np.array_equal(o["height_map"], s["synth_height_map"])

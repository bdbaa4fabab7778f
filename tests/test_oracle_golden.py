"""The oracle is pinned to the real reference: every fixture in tests/golden was
written by oracle/make_golden.py from the unmodified reference package."""

import json

import numpy as np
import pytest

from conftest import load_golden, scene_names
from oracle import crowd as C
from oracle import scene as S
from oracle.rng import PCG64Emu, child_seed, pairwise_sum


def test_child_seeds_match_reference():
    k = load_golden("rng_kat.npz")
    cs = [child_seed(0, "env", i) for i in range(8)] + [
        child_seed(2 ** 64 - 1, "crowd", 12345), child_seed(5, "wfc", 15),
        child_seed(123, "terrain-stage"), child_seed(0)]
    assert np.array_equal(np.array(cs, np.uint64), k["child_seeds"])


@pytest.mark.parametrize("i", range(6))
def test_pcg64_emulator_known_answers(i):
    k = load_golden("rng_kat.npz")
    seed = int(k[f"s{i}_seed"])
    e = PCG64Emu(seed)
    st = [int(v) for v in k[f"s{i}_state"]]
    assert e.state == (st[0] << 64 | st[1]) and e.inc == (st[2] << 64 | st[3])
    assert [e.next64() for _ in range(16)] == [int(v) for v in k[f"s{i}_next64"]]
    e = PCG64Emu(seed)
    seq = []
    for _ in range(64):
        seq += [e.integers(2 ** 63), e.integers(17), e.random() * 2 ** 53,
                e.integers(3, 50000), e.uniform(0.0, 32.0) * 2 ** 40]
    assert np.array_equal(np.array(seq, np.float64), k[f"s{i}_mixed"])
    assert PCG64Emu(seed).permutation(1000) == list(k[f"s{i}_perm"])


def test_pairwise_sum_matches_numpy():
    for n in range(1, 130):
        v = np.random.default_rng(n).uniform(0.0, 1.0, n)
        assert pairwise_sum(v) == v.sum()


@pytest.mark.parametrize("name", scene_names())
def test_scene_oracle_matches_reference(name, catalog):
    g = load_golden(f"scene_{name}.npz")
    spec = json.loads(str(g["spec"]))
    sc = S.generate_scene(dict(seed=spec["seed"], extent=(spec["extent"], spec["extent"]),
                               res=spec["res"], task=spec["task"], split=spec["split"],
                               density=spec["density"], mix=spec["mix"]), catalog)
    assert np.array_equal(sc["zones"], g["zones"])
    assert np.array_equal(sc["assign"], g["assign"])
    assert [t[2] for t in sc["tiles"]] == list(g["tile_code"])
    assert np.array_equal(np.array([t[3] for t in sc["tiles"]]), g["tile_p"])
    assert int(sc["noise_seed"]) == int(g["noise_seed"])
    objs = np.array(sc["objects"], np.float64).reshape(-1, 4)
    assert np.array_equal(objs, g["objects"])
    assert bool(sc["overflow"]) == bool(g["overflow"])
    assert np.array_equal(sc["labels"], g["labels"])
    assert np.array_equal(sc["elev"].view(np.uint32), g["elev"].view(np.uint32))
    near = C.nearest_obstacle_map(sc["labels"])
    if g["nearest"].size:
        assert np.array_equal(near, g["nearest"])
    else:
        assert near is None
    if spec["peds"]:
        sp = C.spawn_agents(sc["labels"], spec["res"], spec["peds"],
                            child_seed(spec["seed"], "crowd", 0))
        assert np.array_equal(sp["pos"], g["spawn_pos"])
        assert np.array_equal(sp["goal"], g["spawn_goal"])
        assert np.array_equal(sp["kind"], g["spawn_kind"])
        assert np.array_equal(sp["pref"], g["spawn_pref"])
        assert np.array_equal(sp["radius"], g["spawn_radius"])


def test_crowd_oracle_trajectory_matches_reference(catalog):
    g = load_golden("crowd_cfg1.npz")
    grids, per_env = [], []
    for i, s in enumerate(g["env_seeds"]):
        s = int(s)
        sc = S.generate_scene(dict(seed=s, extent=(32.0, 32.0), res=0.25, task="NavDynamic",
                                   split="Train", density=20 / 41,
                                   mix={"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}),
                              catalog)
        grids.append((sc["labels"], 0.25))
        per_env.append(C.spawn_agents(sc["labels"], 0.25, 8, child_seed(s, "crowd", 0)))
    f = C.CrowdFieldOracle(grids, C.Config(), [int(s) for s in g["run_seeds"]])
    f.set_agents(per_env)
    for t in range(g["pos"].shape[0]):
        f.step(robot_pos=g["rpos"][t], robot_vel=g["rvel"][t], robot_radius=0.35,
               env_mask=g["mask"][t])
        assert np.array_equal(f.pos, g["pos"][t]), t
        assert np.array_equal(f.vel, g["vel"][t]), t
        assert np.array_equal(f.goal, g["goal"][t]), t
        assert np.array_equal(f.waypoint, g["waypoint"][t]), t
        assert np.array_equal(f.last_gap_by_env, g["gap"][t]), t

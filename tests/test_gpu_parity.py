"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden fixtures and the oracle, bit-exact (integer and float64 outputs)."""

import json

import numpy as np
import pytest

from conftest import golden_catalog, load_golden, scene_names

pytestmark = pytest.mark.gpu

MIX = {"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}


def _spec(d, peds=None):
    from paper_2505_00690_b200.urbangen import SceneSpec, Split, TaskKind
    return SceneSpec(seed=int(d["seed"]), extent_m=(d["extent"], d["extent"]),
                     task_kind=TaskKind(d["task"]), split=Split(d["split"]),
                     object_density=d["density"], pedestrian_count=d["peds"] if peds is None else peds,
                     terrain_mix=d["mix"], grid_resolution_m=d["res"])


def test_device_child_seeds_and_streams(torch_cuda):
    torch = torch_cuda
    from oracle.rng import child_seed
    from paper_2505_00690_b200 import _lib
    from paper_2505_00690_b200.rng import child_seeds_device, seeds_to_tensor
    k = load_golden("rng_kat.npz")
    zero = torch.zeros(8, dtype=torch.int64, device="cuda")
    got = child_seeds_device(zero, "env", torch.arange(8, device="cuda"))
    assert np.array_equal(got.cpu().numpy().view(np.uint64), k["child_seeds"][:8])
    parents = [0, 1, 2 ** 64 - 1, 12345678901234567890]
    pt = seeds_to_tensor(parents, "cuda")
    for lab in ("crowd-run", "crowd", "resample"):
        kk = None if lab == "crowd-run" else torch.tensor([0, 7, 12345, 3], device="cuda")
        d = child_seeds_device(pt, lab, kk).cpu().numpy().view(np.uint64)
        exp = [child_seed(p, lab) if kk is None else child_seed(p, lab, int(x))
               for p, x in zip(parents, [0, 7, 12345, 3])]
        assert [int(v) for v in d] == exp
    seeds = [int(k[f"s{i}_seed"]) for i in range(6)]
    st = torch.empty((6, 48), dtype=torch.uint8, device="cuda")
    _lib.check(_lib.lib().cw_seed_streams(6, _lib.ptr(seeds_to_tensor(seeds, "cuda")), _lib.ptr(st),
                                          _lib.stream_ptr()), "seed")
    raw = st.cpu().numpy().view(np.uint64).reshape(6, 6)
    for i in range(6):
        assert np.array_equal(raw[i, :4], k[f"s{i}_state"]), i


@pytest.mark.parametrize("name", scene_names())
def test_scene_sampling_matches_reference(name, torch_cuda):
    from oracle.rng import child_seed
    from paper_2505_00690_b200.urbangen import SceneSampler
    g = load_golden(f"scene_{name}.npz")
    d = json.loads(str(g["spec"]))
    spec = _spec(d)
    s = SceneSampler(spec, 1)
    b = s.sample([d["seed"]], [child_seed(d["seed"], "crowd", 0)])
    assert np.array_equal(b.zones[0].cpu().numpy(), g["zones"])
    assert np.array_equal(b.assign[0].cpu().numpy(), g["assign"])
    n = int(b.n_tiles[0])
    assert n == len(g["tile_code"])
    assert np.array_equal(b.tile_code[0, :n].cpu().numpy(), g["tile_code"])
    assert np.array_equal(b.tile_kind[0, :n].cpu().numpy(), g["tile_kind"])
    assert np.array_equal(b.tile_p[0, :n].cpu().numpy(), g["tile_p"])
    assert int(b.noise_seed[0]) & (2 ** 64 - 1) == int(g["noise_seed"])
    m = int(b.obj_n[0])
    objs = np.concatenate([b.obj_cat[0, :m].cpu().numpy()[:, None].astype(np.float64),
                           b.obj_pose[0, :m].cpu().numpy()], axis=1)
    assert np.array_equal(objs.reshape(-1, 4), g["objects"])
    assert bool(b.overflow[0]) == bool(g["overflow"])
    assert np.array_equal(b.labels[0].cpu().numpy(), g["labels"])
    assert np.array_equal(b.elev[0].cpu().numpy().view(np.uint32), g["elev"].view(np.uint32))
    if g["nearest"].size:
        assert int(b.has_obs[0]) == 1
        assert np.array_equal(b.nearest[0].cpu().numpy(), g["nearest"])
    else:
        assert int(b.has_obs[0]) == 0
    walk = np.flatnonzero(g["labels"].ravel() == 2)
    assert int(b.walk_n[0]) == walk.size
    assert np.array_equal(b.walk[0, :walk.size].cpu().numpy(), walk)
    if d["peds"]:
        A = d["peds"]
        assert np.array_equal(b.sp_pos[0, :A].cpu().numpy(), g["spawn_pos"])
        assert np.array_equal(b.sp_goal[0, :A].cpu().numpy(), g["spawn_goal"])
        assert np.array_equal(b.sp_kind[0, :A].cpu().numpy(), g["spawn_kind"])
        assert np.array_equal(b.sp_pref[0, :A].cpu().numpy(), g["spawn_pref"])


def test_batch_rows_match_solo_sampling(torch_cuda):
    """Async sampling is row-independent: env i in a batch of 12 == env i alone."""
    from oracle.rng import child_seed
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec, TaskKind
    spec = SceneSpec(seed=0, extent_m=(32.0, 32.0), task_kind=TaskKind.NAV_DYNAMIC,
                     object_density=20 / 41, pedestrian_count=8, terrain_mix=MIX,
                     grid_resolution_m=0.25)
    seeds = [child_seed(9, "env", i) for i in range(12)]
    cs = [child_seed(s, "crowd", 0) for s in seeds]
    big = SceneSampler(spec, 12).sample(seeds, cs)
    for i in (0, 5, 11):
        solo = SceneSampler(spec, 1).sample([seeds[i]], [cs[i]])
        for name in ("labels", "elev", "nearest", "sp_pos", "sp_goal", "assign"):
            assert np.array_equal(getattr(big, name)[i].cpu().numpy(),
                                  getattr(solo, name)[0].cpu().numpy()), (i, name)


def _device_crowd(seeds, spec_kw, peds):
    from oracle.rng import child_seed
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec, TaskKind
    spec = SceneSpec(seed=0, task_kind=TaskKind.NAV_DYNAMIC, pedestrian_count=peds,
                     terrain_mix=MIX, **spec_kw)
    b = SceneSampler(spec, len(seeds)).sample(seeds, [child_seed(s, "crowd", 0) for s in seeds])
    f = CrowdField(b, CrowdConfig(), [child_seed(s, "crowd-run") for s in seeds])
    f.set_from_spawn(b)
    return b, f


def test_crowd_trajectory_matches_reference_golden(torch_cuda):
    """60 ticks of CrowdField.step on cfg1-shape envs (obstacles, robot lane,
    env_mask, goal resampling): bit-exact against the reference's trajectory."""
    g = load_golden("crowd_cfg1.npz")
    seeds = [int(s) for s in g["env_seeds"]]
    b, f = _device_crowd(seeds, dict(extent_m=(32.0, 32.0), object_density=20 / 41,
                                     grid_resolution_m=0.25), 8)
    for t in range(g["pos"].shape[0]):
        f.step(robot_pos=g["rpos"][t], robot_vel=g["rvel"][t], robot_radius=0.35,
               env_mask=g["mask"][t])
        assert np.array_equal(f.pos, g["pos"][t]), t
        assert np.array_equal(f.vel, g["vel"][t]), t
        assert np.array_equal(f.goal, g["goal"][t]), t
        assert np.array_equal(f.waypoint, g["waypoint"][t]), t
        assert np.array_equal(f.last_gap_by_env, g["gap"][t]), t


@pytest.mark.parametrize("shape", ["cfg1", "cfg2"])
def test_crowd_matches_oracle(shape, torch_cuda):
    from oracle import crowd as C
    from oracle.rng import child_seed
    if shape == "cfg1":
        kw, peds, E, T = dict(extent_m=(32.0, 32.0), object_density=20 / 41, grid_resolution_m=0.25), 8, 6, 40
    else:
        kw, peds, E, T = dict(extent_m=(32.0, 32.0), object_density=64 / 41, grid_resolution_m=0.125), 32, 2, 25
    seeds = [child_seed(77, "env", i) for i in range(E)]
    b, f = _device_crowd(seeds, kw, peds)
    grids = [(b.labels[i].cpu().numpy(), kw["grid_resolution_m"]) for i in range(E)]
    agents = []
    for i, s in enumerate(seeds):
        sp = C.spawn_agents(grids[i][0], kw["grid_resolution_m"], peds, child_seed(s, "crowd", 0))
        assert np.array_equal(sp["pos"], b.sp_pos[i].cpu().numpy())
        agents.append(sp)
    ref = C.CrowdFieldOracle(grids, C.Config(), [child_seed(s, "crowd-run") for s in seeds])
    ref.set_agents(agents)
    rng = np.random.default_rng(1)
    for t in range(T):
        rp = rng.uniform(2.0, 30.0, (E, 2))
        rv = rng.uniform(-1.0, 1.0, (E, 2))
        f.step(robot_pos=rp, robot_vel=rv)
        ref.step(robot_pos=rp, robot_vel=rv)
        assert np.array_equal(f.pos, ref.pos), t
        assert np.array_equal(f.vel, ref.vel), t
        assert np.array_equal(f.goal, ref.goal), t


@pytest.mark.parametrize("arena,E,A,T", [(12.0, 4, 40, 150), (24.0, 2, 200, 60)])
def test_dense_open_grid_fallback_matches_oracle(arena, E, A, T, torch_cuda):
    """Obstacle-free dense crowds exercise the least-violation fallback and the
    stall retry heavily (acceptance sweep shape, tests/test_acceptance.py:209-249).
    A = 200 runs the cell-binned neighbour search (A >= 128)."""
    from oracle import crowd as C
    from paper_2505_00690_b200.crowd import CrowdAgent, CrowdConfig, CrowdField
    from paper_2505_00690_b200.urbangen import OccupancyGrid
    res = 0.1
    n = int(arena / res)
    labels = np.full((n, n), 2, np.uint8)
    occ = OccupancyGrid(res, labels, np.zeros((n, n), np.float32))
    lists = []
    for e in range(E):
        r = np.random.default_rng(e)
        lst = []
        for a in range(A):
            while True:
                p = r.uniform(1.5, arena - 1.5, 2)
                if all(np.hypot(*(p - o.position)) > 0.7 for o in lst):
                    break
            lst.append(CrowdAgent(id=a, position=p, velocity=np.zeros(2), radius=0.3,
                                  preferred_speed=float(r.uniform(0.8, 1.4)),
                                  goal=r.uniform(1.5, arena - 1.5, 2)))
        lists.append(lst)
    cfg = CrowdConfig(safety_margin=0.05)
    f = CrowdField([occ] * E, cfg, [5000 + e for e in range(E)])
    f.set_agents(lists)
    ref = C.CrowdFieldOracle([(labels, res)] * E, C.Config(safety_margin=0.05), [5000 + e for e in range(E)])
    ref.set_agents([dict(pos=np.array([a.position for a in l]), goal=np.array([a.goal for a in l]),
                         radius=np.full(A, 0.3), pref=np.array([a.preferred_speed for a in l]),
                         max_speed=np.full(A, 2.0), kind=np.zeros(A, np.int8)) for l in lists])
    for t in range(T):
        f.step()
        ref.step()
        assert np.array_equal(f.pos, ref.pos), t
        assert np.array_equal(f.vel, ref.vel), t
        assert np.array_equal(f.last_gap_by_env, ref.last_gap_by_env), t
    assert f.stats()["lp_fallbacks"] > 0


def test_head_on_pair_mirrors_and_passes(torch_cuda):
    """tests/test_crowd.py:243-265 on the device path."""
    from paper_2505_00690_b200.crowd import CrowdAgent, CrowdConfig, CrowdField
    from paper_2505_00690_b200.urbangen import OccupancyGrid
    n = 300
    occ = OccupancyGrid(0.1, np.full((n, n), 2, np.uint8), np.zeros((n, n), np.float32))
    a = CrowdAgent(id=0, position=np.array([10.0, 15.0]), velocity=np.array([1.0, 0.0]),
                   radius=0.3, preferred_speed=1.0, goal=np.array([20.0, 15.0]))
    b = CrowdAgent(id=1, position=np.array([20.0, 15.0]), velocity=np.array([-1.0, 0.0]),
                   radius=0.3, preferred_speed=1.0, goal=np.array([10.0, 15.0]))
    f = CrowdField([occ], CrowdConfig(), [0], resample_goals=False)
    f.set_agents([[a, b]])
    passed, min_d = False, np.inf
    for _ in range(500):
        f.step()
        p = f.pos[0]
        v = f.vel[0]
        assert np.abs((p[0] - 15.0) + (p[1] - 15.0)).max() < 1e-9
        assert np.abs(v[0] + v[1]).max() < 1e-9
        min_d = min(min_d, float(np.hypot(*(p[0] - p[1]))))
        if p[0, 0] > p[1, 0] + 0.3:
            passed = True
            break
    assert passed and min_d >= 0.6 - 1e-9


def test_batched_env_resample_slots(torch_cuda):
    """BatchedEnv.resample: touched rows change, others do not; a resampled row
    equals a fresh sample with the reference's resample seed (batch.py:326-339)."""
    from oracle.rng import child_seed
    from paper_2505_00690_b200.envcore import BatchedEnv, Scheme
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec, TaskKind
    spec = SceneSpec(seed=0, extent_m=(32.0, 32.0), task_kind=TaskKind.NAV_DYNAMIC,
                     object_density=20 / 41, pedestrian_count=8, terrain_mix=MIX,
                     grid_resolution_m=0.25)
    env = BatchedEnv(spec, Scheme.ASYNC, master_seed=3, k=6)
    before = env.labels_stack.clone()
    env.resample([1, 4])
    after = env.labels_stack
    for i in range(6):
        same = bool((before[i] == after[i]).all())
        assert same == (i not in (1, 4)), i
    s4 = child_seed(env.env_seeds[4], "resample", 1)
    solo = SceneSampler(spec, 1).sample([s4], [child_seed(env.env_seeds[4], "crowd", 1)])
    assert np.array_equal(solo.labels[0].cpu().numpy(), after[4].cpu().numpy())
    assert np.array_equal(solo.sp_pos[0].cpu().numpy(), env.crowd.pos_t[4].cpu().numpy())
    env.step_crowd()


def test_shard_invariance_sampling_and_crowd(torch_cuda):
    """W=1 vs W=2: global env ids [0,6) in one batch equal the two
    shards [0,3) + [3,6) run as separate batches, over sampling and 20 ticks."""
    import torch
    from paper_2505_00690_b200 import shard
    seeds_all = shard.env_seeds(0, shard.env_ids(0, 1, 6))
    kw = dict(extent_m=(32.0, 32.0), object_density=20 / 41, grid_resolution_m=0.25)
    rp = np.random.default_rng(3).uniform(3.0, 29.0, (20, 6, 2))
    b1, f1 = _device_crowd(seeds_all, kw, 8)
    parts = []
    for r in range(2):
        ids = shard.env_ids(r, 2, 3)
        parts.append(_device_crowd(shard.env_seeds(0, ids), kw, 8))
    for t in range(20):
        f1.step(robot_pos=rp[t], robot_vel=np.zeros((6, 2)))
        for r, (_, f) in enumerate(parts):
            f.step(robot_pos=rp[t, 3 * r:3 * r + 3], robot_vel=np.zeros((3, 2)))
    for r, (b, f) in enumerate(parts):
        sl = slice(3 * r, 3 * r + 3)
        assert np.array_equal(b1.labels[sl].cpu().numpy(), b.labels.cpu().numpy())
        assert np.array_equal(f1.pos[sl], f.pos)
        assert np.array_equal(f1.vel[sl], f.vel)
        assert np.array_equal(f1.goal[sl], f.goal)
        # the bench's per-env state checksum: on device == on host, and shard-invariant
        c_dev = shard.state_checksum(f.pos_t, f.vel_t, f.goal_t).cpu()
        assert torch.equal(c_dev, shard.state_checksum(f.pos, f.vel, f.goal))
        assert torch.equal(c_dev, shard.state_checksum(f1.pos_t, f1.vel_t, f1.goal_t).cpu()[sl])


@pytest.mark.parametrize("peds", [96, 160])
def test_blocks_layout_dense_crowd_matches_oracle(peds, torch_cuda):
    """cfg4 shape (block layout with roads/crosswalks, NavClear placement, many
    pedestrians, neighbor_distance 3 m) against the oracle for a few ticks;
    160 pedestrians run the cell-binned neighbour search."""
    from oracle import crowd as C
    from oracle import scene as S
    from oracle.rng import child_seed
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec, TaskKind
    seed = child_seed(0, "env", 11)
    spec = SceneSpec(seed=seed, extent_m=(48.0, 48.0), task_kind=TaskKind.NAV_CLEAR,
                     object_density=0.0, pedestrian_count=peds, terrain_mix=MIX,
                     grid_resolution_m=0.25)
    b = SceneSampler(spec, 1).sample([seed], [child_seed(seed, "crowd", 0)])
    sc = S.generate_scene(dict(seed=seed, extent=(48.0, 48.0), res=0.25, task="NavClear",
                               split="Train", density=0.0, mix=MIX), golden_catalog())
    assert np.array_equal(b.zones[0].cpu().numpy(), sc["zones"])
    assert np.array_equal(b.labels[0].cpu().numpy(), sc["labels"])
    sp = C.spawn_agents(sc["labels"], 0.25, peds, child_seed(seed, "crowd", 0))
    assert np.array_equal(b.sp_pos[0].cpu().numpy(), sp["pos"])
    assert np.array_equal(b.sp_goal[0].cpu().numpy(), sp["goal"])
    run = [child_seed(seed, "crowd-run")]
    f = CrowdField(b, CrowdConfig(neighbor_distance=3.0), run)
    f.set_from_spawn(b)
    ref = C.CrowdFieldOracle([(sc["labels"], 0.25)], C.Config(neighbor_distance=3.0), run)
    ref.set_agents([sp])
    rng = np.random.default_rng(4)
    for t in range(4):
        rp = rng.uniform(5.0, 43.0, (1, 2))
        f.step(robot_pos=rp, robot_vel=np.zeros((1, 2)))
        ref.step(robot_pos=rp, robot_vel=np.zeros((1, 2)))
        assert np.array_equal(f.pos, ref.pos), t
        assert np.array_equal(f.vel, ref.vel), t


@pytest.mark.parametrize("ext,res,task,peds", [((13.3, 17.7), 0.1, "NavStatic", 5),
                                              ((21.0, 9.5), 0.25, "NavDynamic", 6),
                                              ((44.0, 40.5), 0.5, "NavStatic", 12),
                                              ((30.0, 12.0), 0.2, "Traverse", 4)])
def test_odd_shaped_scenes_match_oracle(ext, res, task, peds, torch_cuda):
    """Non-square grids whose width is not a multiple of 4, block and strip
    layouts, Traverse regions: every sampling output bit-exact vs the oracle."""
    from oracle import crowd as C
    from oracle import scene as S
    from oracle.rng import child_seed
    from paper_2505_00690_b200.urbangen import SceneSampler, SceneSpec, TaskKind
    mix = {"Flat": 0.3, "Slope": 0.3, "Stair": 0.2, "Rough": 0.2}
    for i in range(2):
        seed = child_seed(31, "env", i)
        spec = SceneSpec(seed=seed, extent_m=ext, task_kind=TaskKind(task), object_density=1.0,
                         pedestrian_count=peds, terrain_mix=mix, grid_resolution_m=res)
        b = SceneSampler(spec, 1).sample([seed], [child_seed(seed, "crowd", 0)])
        sc = S.generate_scene(dict(seed=seed, extent=ext, res=res, task=task, split="Train",
                                   density=1.0, mix=mix), golden_catalog())
        assert np.array_equal(b.zones[0].cpu().numpy(), sc["zones"])
        assert np.array_equal(b.assign[0].cpu().numpy(), sc["assign"])
        assert np.array_equal(b.labels[0].cpu().numpy(), sc["labels"])
        assert np.array_equal(b.elev[0].cpu().numpy().view(np.uint32), sc["elev"].view(np.uint32))
        m = int(b.obj_n[0])
        assert m == len(sc["objects"])
        near = C.nearest_obstacle_map(sc["labels"])
        if near is not None:
            assert np.array_equal(b.nearest[0].cpu().numpy(), near)
        if task != "Traverse":   # traverse spawn uses the segment mask (batch.py:174-176)
            sp = C.spawn_agents(sc["labels"], res, peds, child_seed(seed, "crowd", 0))
            assert np.array_equal(b.sp_pos[0, :peds].cpu().numpy(), sp["pos"])
            assert np.array_equal(b.sp_goal[0, :peds].cpu().numpy(), sp["goal"])

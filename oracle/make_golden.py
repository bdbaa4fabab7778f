"""Generate tests/golden/*.npz from the REAL reference (build container only).

Run:  PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py
It imports the unmodified reference from /root/reference/pkg/src (read-only),
drives its public entry points (generate_scene, rasterize_occupancy,
spawn_agents, CrowdField, numpy Generator) and stores their outputs.  The
fixtures travel with the repo; /root/reference does not (tests never read it).
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
MIX = {"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}

# (name, seed, extent, res, task, density, split, mix, peds)
SCENES = [
    ("cfg1_e0", ("env", 0), 32.0, 0.25, "NavDynamic", 20 / 41, "Train", MIX, 8),
    ("cfg1_e1", ("env", 1), 32.0, 0.25, "NavDynamic", 20 / 41, "Train", MIX, 8),
    ("cfg1_e2", ("env", 2), 32.0, 0.25, "NavDynamic", 20 / 41, "Train", MIX, 8),
    ("cfg1_e3", ("env", 3), 32.0, 0.25, "NavDynamic", 20 / 41, "Train", MIX, 8),
    ("cfg2_e0", ("env", 0), 32.0, 0.125, "NavDynamic", 64 / 41, "Train", MIX, 32),
    ("static10_s11", 11, 10.0, 0.1, "NavStatic", 1.0, "Train", None, 0),
    ("test15_s5", 5, 15.0, 0.1, "NavStatic", 1.0, "Test", MIX, 4),
    ("blocks48_s3", 3, 48.0, 0.25, "NavStatic", 0.5, "Train", MIX, 16),
    ("clear64_e2", ("env", 2), 64.0, 0.5, "NavClear", 0.0, "Train", MIX, 24),
]


def _scene_arrays(spec, peds, child_seed):
    from citywalk.crowd import spawn_agents
    from citywalk.crowd.field import _nearest_obstacle_map
    from citywalk.urbangen import generate_scene, rasterize_occupancy
    from citywalk.urbangen.catalog import load_catalog

    names = [e.category for e in load_catalog()]
    sc = generate_scene(spec)
    occ = rasterize_occupancy(sc)
    tiles = sc.terrain.tiles
    code = {"corner": 0, "rough": 3}
    tcode, tp, kind, param = [], [], [], []
    kinds = ["Flat", "SlopeUp", "SlopeDown", "StairUp", "StairDown", "Rough"]
    for t in tiles:
        s = t.shape
        if s["type"] == "stair":
            tcode.append(1 if s["axis"] == "u" else 2)
            tp.append([s["a"], s["b"], 0.0, 0.0])
        elif s["type"] == "corner":
            tcode.append(0)
            tp.append(list(s["h"]))
        else:
            tcode.append(code["rough"])
            tp.append([s["base"], s["amp"], 0.0, 0.0])
        kind.append(kinds.index(t.kind.value))
        param.append(t.param)
    objs = np.array([[names.index(o.category), o.x, o.y, o.yaw] for o in sc.objects]
                    ).reshape(-1, 4)
    near = _nearest_obstacle_map(occ.labels)
    out = dict(
        zones=sc.zones.grid, assign=sc.terrain.assignment,
        tile_code=np.array(tcode, np.int8), tile_p=np.array(tp), tile_kind=np.array(kind, np.int8),
        tile_param=np.array(param), noise_seed=np.uint64(sc.terrain.noise_seed),
        objects=objs, overflow=np.bool_(sc.placement_overflow),
        labels=occ.labels, elev=occ.elevation,
        nearest=(near if near is not None else np.zeros((0, 0), np.int64)),
    )
    if peds:
        ag = spawn_agents(occ, peds, child_seed(spec.seed, "crowd", 0))
        out.update(
            spawn_pos=np.array([a.position for a in ag]), spawn_goal=np.array([a.goal for a in ag]),
            spawn_kind=np.array([int(a.kind) for a in ag], np.int8),
            spawn_pref=np.array([a.preferred_speed for a in ag]),
            spawn_radius=np.array([a.radius for a in ag]),
        )
    return out


def main():
    sys.path.insert(0, REF)
    from citywalk.crowd import CrowdConfig, CrowdField, spawn_agents
    from citywalk.rng import child_seed
    from citywalk.urbangen import SceneSpec, Split, TaskKind, generate_scene, rasterize_occupancy
    from citywalk.urbangen.catalog import load_catalog

    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "catalog.json"), "w") as fh:
        json.dump([e.to_dict() for e in load_catalog()], fh, indent=1)

    # --- RNG known answers (numpy Generator(PCG64) as the reference calls it)
    kat = {}
    for k, s in enumerate([0, 1, 2 ** 32 + 7, 12345678901234567890,
                           child_seed(0, "env", 0), child_seed(7, "crowd-run")]):
        g = np.random.Generator(np.random.PCG64(s))
        st = g.bit_generator.state["state"]
        kat[f"s{k}_seed"] = np.uint64(s)
        kat[f"s{k}_state"] = np.array([st["state"] >> 64, st["state"] & (2 ** 64 - 1),
                                       st["inc"] >> 64, st["inc"] & (2 ** 64 - 1)], np.uint64)
        kat[f"s{k}_next64"] = g.bit_generator.random_raw(16).astype(np.uint64)
        g = np.random.Generator(np.random.PCG64(s))
        seq = []
        for i in range(64):   # interleaved draw kinds: exercises the 32-bit half buffer
            seq += [g.integers(2 ** 63), g.integers(17), g.random() * 2 ** 53,
                    g.integers(3, 50000), g.uniform(0.0, 32.0) * 2 ** 40]
        kat[f"s{k}_mixed"] = np.array(seq, np.float64)
        kat[f"s{k}_perm"] = np.random.Generator(np.random.PCG64(s)).permutation(1000)
    cs = [child_seed(0, "env", i) for i in range(8)] + [
        child_seed(2 ** 64 - 1, "crowd", 12345), child_seed(5, "wfc", 15),
        child_seed(123, "terrain-stage"), child_seed(0)]
    kat["child_seeds"] = np.array(cs, np.uint64)
    np.savez_compressed(os.path.join(OUT, "rng_kat.npz"), **kat)

    # --- scenes
    for name, seed, ext, res, task, dens, split, mix, peds in SCENES:
        if isinstance(seed, tuple):
            seed = child_seed(0, *seed)
        spec = SceneSpec(seed=seed, extent_m=(ext, ext), task_kind=TaskKind(task),
                         split=Split(split), object_density=dens, pedestrian_count=peds,
                         **({"terrain_mix": mix} if mix else {}), grid_resolution_m=res)
        arr = _scene_arrays(spec, peds, child_seed)
        arr["spec"] = np.array(json.dumps(dict(seed=seed, extent=ext, res=res, task=task,
                                               density=dens, split=split, mix=mix or spec.terrain_mix,
                                               peds=peds)))
        np.savez_compressed(os.path.join(OUT, f"scene_{name}.npz"), **arr)

    # --- crowd trajectory (cfg1 shape: 4 envs x 8 peds, obstacles, robot lane)
    E, T = 4, 60
    occs, seeds, lists = [], [], []
    for i in range(E):
        s = child_seed(0, "env", i)
        spec = SceneSpec(seed=s, extent_m=(32.0, 32.0), task_kind=TaskKind.NAV_DYNAMIC,
                         object_density=20 / 41, pedestrian_count=8, terrain_mix=MIX,
                         grid_resolution_m=0.25)
        occ = rasterize_occupancy(generate_scene(spec))
        occs.append(occ)
        seeds.append(s)
        lists.append(spawn_agents(occ, 8, child_seed(s, "crowd", 0)))
    run_seeds = [child_seed(s, "crowd-run") for s in seeds]
    field = CrowdField(occs, CrowdConfig(), env_seeds=run_seeds)
    field.set_agents(lists)
    rng = np.random.default_rng(2026)
    rpos = rng.uniform(4.0, 28.0, (T, E, 2))
    rvel = rng.uniform(-1.0, 1.0, (T, E, 2))
    mask = rng.random((T, E)) < 0.9
    P, V, G, W, gap = [], [], [], [], []
    for t in range(T):
        field.step(robot_pos=rpos[t], robot_vel=rvel[t], robot_radius=0.35, env_mask=mask[t])
        P.append(field.pos.copy())
        V.append(field.vel.copy())
        G.append(field.goal.copy())
        W.append(field.waypoint.copy())
        gap.append(field.last_gap_by_env.copy())
    np.savez_compressed(
        os.path.join(OUT, "crowd_cfg1.npz"),
        env_seeds=np.array(seeds, np.uint64), run_seeds=np.array(run_seeds, np.uint64),
        rpos=rpos, rvel=rvel, mask=mask, pos=np.array(P), vel=np.array(V), goal=np.array(G),
        waypoint=np.array(W), gap=np.array(gap))
    print("golden fixtures written to", os.path.normpath(OUT))


if __name__ == "__main__":
    main()

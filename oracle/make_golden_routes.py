"""Generate tests/golden/routes.npz from the REAL reference (build container only).

Run:  PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_routes.py
Stores scene.routes (urbangen/scene.py:102-158, _sample_route_anchors) for a set
of seeded specs (courtyard, block, traverse layouts; several resolutions), the
spawn pose BatchedEnv._spawn draws from them (batch.py:183-198), and the
clearance field chamfer_distance(~walkable) (gridmath.py:8-39).
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
MIX = {"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}

# (seed label/int, extent, res, task, density)
CASES = ([(("env", i), 32.0, 0.25, "NavDynamic", 20 / 41) for i in range(12)] +
         [(("env", i), 32.0, 0.125, "NavDynamic", 64 / 41) for i in range(3)] +
         [(3, 48.0, 0.25, "NavStatic", 0.5), (7, 48.0, 0.25, "NavClear", 0.0),
          (11, 10.0, 0.1, "NavStatic", 1.0), (5, 15.0, 0.1, "NavStatic", 1.0),
          (21, 24.0, 0.2, "Traverse", 0.5), (22, 20.0, 0.25, "Traverse", 1.0)])


def main():
    sys.path.insert(0, REF)
    from citywalk.gridmath import chamfer_distance
    from citywalk.rng import child_seed, make_rng
    from citywalk.urbangen import SceneSpec, TaskKind, generate_scene, rasterize_occupancy
    out = {}
    for n, (seed, ext, res, task, dens) in enumerate(CASES):
        if isinstance(seed, tuple):
            seed = child_seed(0, *seed)
        spec = SceneSpec(seed=seed, extent_m=(ext, ext), task_kind=TaskKind(task), object_density=dens,
                         pedestrian_count=0, terrain_mix=MIX, grid_resolution_m=res)
        sc = generate_scene(spec)
        occ = rasterize_occupancy(sc)
        walk = occ.labels == 2
        clear = chamfer_distance(~walk, res)
        routes = np.array(sc.routes, np.float64).reshape(-1, 2, 2)
        spawn = []
        for rc in range(3):   # BatchedEnv._spawn pick for reset counts 0..2 (env_seed = seed)
            rng = make_rng(seed, "spawn", rc)
            spawn.append(int(rng.integers(len(sc.routes))))
        out[f"c{n}_spec"] = np.array(json.dumps(dict(seed=seed, extent=ext, res=res, task=task, density=dens)))
        out[f"c{n}_labels"] = occ.labels
        out[f"c{n}_clearance"] = clear
        out[f"c{n}_routes"] = routes
        out[f"c{n}_spawn_pick"] = np.array(spawn, np.int64)
        print(n, task, ext, res, len(sc.routes))
    out["n"] = np.int64(len(CASES))
    np.savez_compressed(os.path.join(OUT, "routes.npz"), **out)


if __name__ == "__main__":
    main()

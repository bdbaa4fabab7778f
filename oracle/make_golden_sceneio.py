"""Generate tests/golden/sceneio.json from the REAL reference (build container only).

Run:  PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_sceneio.py
Stores, for seeded specs over every layout (courtyard, block grids, traverse
strip; Train/Test splits; several resolutions and terrain mixes):
  * scene_hash(generate_scene(spec))                  (urbangen/scene.py:229-230)
  * the canonical JSON text of the small scenes        (scene.py:206-207, jsonio.py:29-39)
and BatchedEnv.scene_hashes for Async / Sync batches, including after a
resampling reset (envcore/batch.py:126-131, 326-339).
"""

import json
import os
import sys

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
MIX = {"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}
MIX2 = {"Flat": 0.7, "Slope": 0.1, "Stair": 0.0, "Rough": 0.2}

# (seed label/int, extent, res, task, density, split, mix, keep_json)
CASES = ([(("env", i), 32.0, 0.25, "NavDynamic", 20 / 41, "Train", MIX, i < 2) for i in range(6)] +
         [(("env", i), 32.0, 0.125, "NavDynamic", 64 / 41, "Train", MIX, False) for i in range(2)] +
         [(3, 48.0, 0.25, "NavStatic", 0.5, "Train", MIX, True),
          (7, 48.0, 0.25, "NavClear", 0.0, "Train", MIX, False),
          (9, 64.0, 0.5, "NavDynamic", 0.3, "Test", MIX, True),
          (11, 10.0, 0.1, "NavStatic", 1.0, "Train", MIX2, True),
          (5, 15.0, 0.1, "NavStatic", 1.0, "Test", MIX2, False),
          (21, 24.0, 0.2, "Traverse", 0.5, "Train", MIX, True),
          (22, 20.0, 0.25, "Traverse", 1.0, "Test", MIX2, False),
          (13, 16.0, 0.25, "NavDynamic", 1.0, "Train", {"Flat": 1.0}, True)])


def main():
    sys.path.insert(0, REF)
    from citywalk.envcore import BatchedEnv, Scheme
    from citywalk.rng import child_seed
    from citywalk.urbangen import SceneSpec, Split, TaskKind, generate_scene, scene_hash, scene_to_json
    cases = []
    for n, (seed, ext, res, task, dens, split, mix, keep) in enumerate(CASES):
        if isinstance(seed, tuple):
            seed = child_seed(0, *seed)
        spec = SceneSpec(seed=seed, extent_m=(ext, ext), task_kind=TaskKind(task), split=Split(split),
                         object_density=dens, pedestrian_count=0, terrain_mix=mix, grid_resolution_m=res)
        sc = generate_scene(spec)
        rec = dict(spec=spec.to_dict(), hash=scene_hash(sc))
        if keep:
            rec["json"] = scene_to_json(sc)
        cases.append(rec)
        print(n, task, ext, res, rec["hash"][:12], len(scene_to_json(sc)))
    spec = SceneSpec(seed=0, extent_m=(16.0, 16.0), task_kind=TaskKind.NAV_DYNAMIC, object_density=1.0,
                     pedestrian_count=4, terrain_mix=MIX, grid_resolution_m=0.25)
    envs = {}
    for scheme in (Scheme.ASYNC, Scheme.SYNC):
        env = BatchedEnv(spec, scheme, master_seed=0, k=4)
        envs[scheme.value] = list(env.scene_hashes)
    env = BatchedEnv(spec, Scheme.ASYNC, master_seed=0, k=4)
    env.reset(1, resample=True)
    env.reset(1, resample=False)
    env.reset(1, resample=True)
    envs["Async_resampled"] = list(env.scene_hashes)
    envs["batch_spec"] = spec.to_dict()
    with open(os.path.join(OUT, "sceneio.json"), "w", encoding="utf-8") as fh:
        json.dump(dict(cases=cases, batched=envs), fh, indent=0, sort_keys=True)
        fh.write("\n")


if __name__ == "__main__":
    main()

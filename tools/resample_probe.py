"""cfg5's per-tick re-sampling in isolation: SceneSampler.sample(rows) + set_from_spawn
for the Bernoulli(0.02) rows of a tick, device time (events) and host wall time.
python tools/resample_probe.py [config] [reps]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField  # noqa: E402
from paper_2505_00690_b200.rng import child_seeds_device  # noqa: E402
from paper_2505_00690_b200.urbangen import SceneSampler  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
bench.CFG.clear()
bench.CFG.update(bench.CONFIGS[cfg])
E = bench.CFG["envs"]
dev = torch.device("cuda")
zero = torch.zeros(E, dtype=torch.int64, device=dev)
env = child_seeds_device(zero, "env", torch.arange(E, device=dev))
s = SceneSampler(bench.make_spec(), E)
s.sample(env, child_seeds_device(env, "crowd", 0))
b = s.batch
seeds = [int(x) for x in child_seeds_device(env, "crowd-run").cpu().numpy().view(np.uint64)]
f = CrowdField(b, CrowdConfig(neighbor_distance=bench.CFG["nd"]), seeds)
f.set_from_spawn(b)
rng = np.random.default_rng(0)
counts = torch.zeros(E, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream()
for mode in ("sample", "sample+spawn"):
    dts, walls = [], []
    for k in range(reps):
        rows = np.flatnonzero(rng.random(E) < bench.CFG["resample"])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sl = torch.from_numpy(rows).to(dev)
        counts[sl] += 1
        s.sample(child_seeds_device(env[sl], "resample", counts[sl]), child_seeds_device(env[sl], "crowd", counts[sl]),
                 slots=sl, check=False)
        if mode == "sample+spawn":
            f.set_from_spawn(b, rows=sl)
        e1.record(st)
        torch.cuda.synchronize()
        walls.append(1e3 * (time.perf_counter() - t0))
        dts.append(e0.elapsed_time(e1))
    print(f"{cfg} {mode}: {len(rows)} rows, device {np.median(dts):.2f} ms, wall {np.median(walls):.2f} ms")

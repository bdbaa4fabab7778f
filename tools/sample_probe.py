"""Scene sampling throughput for a bench config with different route chunk sizes (GPU).
Usage: python tools/sample_probe.py [config] [chunk,...]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2505_00690_b200 import _lib  # noqa: E402
from paper_2505_00690_b200.rng import child_seeds_device  # noqa: E402
from paper_2505_00690_b200.urbangen import SceneSampler  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
chunks = [int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "296").split(",")]
bench.CFG.clear()
bench.CFG.update(bench.CONFIGS[cfgname])
E = int(os.environ.get("PROBE_ENVS", bench.CFG["envs"]))
dev = torch.device("cuda")
_lib.build()
spec = bench.make_spec()
env_seeds = child_seeds_device(torch.zeros(E, dtype=torch.int64, device=dev), "env", torch.arange(E, device=dev))
crowd_seeds = child_seeds_device(env_seeds, "crowd", 0)
s = SceneSampler(spec, E, device=dev)
ref = None
for ch in chunks:
    s.route_chunk = ch
    s.batch.route_scratch = None
    s.sample(env_seeds, crowd_seeds, check=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        s.sample(env_seeds, crowd_seeds, check=False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    r = s.batch.routes.cpu().numpy().copy()
    same = ref is None or np.array_equal(r, ref)
    ref = r if ref is None else ref
    print(f"{cfgname} E={E} route_chunk {ch}: {ms:.2f} ms per batch, {E / ms * 1e3:,.0f} scenes/s, routes same {same}")

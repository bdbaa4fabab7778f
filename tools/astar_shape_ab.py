"""Synchronous tick time vs the A* launch shape (search warps per SM: 1 = latency
shape with the larger shared tile pool, 4 = throughput shape) on a bench config."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField  # noqa: E402
from paper_2505_00690_b200.rng import child_seeds_device  # noqa: E402
from paper_2505_00690_b200.urbangen import SceneSampler  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 30
bench.CFG.clear()
bench.CFG.update(bench.CONFIGS[cfg])
C = bench.CFG
E = C["envs"]
dev = torch.device("cuda")
nx = int(np.ceil(C["extent"] / C["res"]))
zero = torch.zeros(E, dtype=torch.int64, device=dev)
env = child_seeds_device(zero, "env", torch.arange(E, device=dev))
b = SceneSampler(bench.make_spec(), E).sample(env, child_seeds_device(env, "crowd", 0))
seeds = [int(x) for x in child_seeds_device(env, "crowd-run").cpu().numpy().view(np.uint64)]
pick = (bench.robot_picks(E, 0).to(dev) * b.walk_n.double()).long()
cell = b.walk.gather(1, pick[:, None])[:, 0].long()
rp = torch.stack([((cell % nx).double() + 0.5) * C["res"], ((cell // nx).double() + 0.5) * C["res"]], 1).contiguous()
rv = torch.zeros_like(rp)
st = torch.cuda.current_stream()
fields = {}
for w in (1, int(os.environ.get("AB_W", "4"))):
    f = CrowdField(b, CrowdConfig(neighbor_distance=C["nd"]), seeds, astar_warps=w)
    f.set_from_spawn(b)
    for _ in range(20):
        f.step(rp, rv, 0.35, check=False)
    fields[w] = f
res = {w: [] for w in fields}
for t in range(T):
    for w, f in fields.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        f.step(rp, rv, 0.35, check=False)
        e1.record(st)
        torch.cuda.synchronize()
        res[w].append(e0.elapsed_time(e1))
assert all(torch.equal(fields[1].pos_t, f.pos_t) for f in fields.values())
print(cfg, {w: round(float(np.mean(v)), 3) for w, v in res.items()}, "ms/tick (astar warps per SM)")

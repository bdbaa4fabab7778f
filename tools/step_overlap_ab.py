"""A/B of the synchronous tick's shape at a bench config: phases 7 (k_orca of the envs
without replans overlapped with k_astar on a second stream) vs phases 1, 2, 4 in order.
Both fields start from the same state and stay bit-identical (checked)."""
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

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 60
bench.CFG.clear()
bench.CFG.update(bench.CONFIGS[cfg])
C = bench.CFG
E = C["envs"]
dev = torch.device("cuda")
nx = int(np.ceil(C["extent"] / C["res"]))
zero = torch.zeros(E, dtype=torch.int64, device=dev)
env = child_seeds_device(zero, "env", torch.arange(E, device=dev))
s = SceneSampler(bench.make_spec(), E)
b = s.sample(env, child_seeds_device(env, "crowd", 0))
run_seeds = [int(x) for x in child_seeds_device(env, "crowd-run").cpu().numpy().view(np.uint64)]
pick = (bench.robot_picks(E, 0).to(dev) * b.walk_n.double()).long()
cell = b.walk.gather(1, pick[:, None])[:, 0].long()
rp = torch.stack([((cell % nx).double() + 0.5) * C["res"], ((cell // nx).double() + 0.5) * C["res"]], 1).contiguous()
rv = torch.zeros_like(rp)
fields = []
for _ in range(2):
    f = CrowdField(b, CrowdConfig(neighbor_distance=C["nd"]), run_seeds)
    f.set_from_spawn(b)
    for _ in range(20):
        f.step(rp, rv, 0.35, check=False)
    fields.append(f)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
st = torch.cuda.current_stream()
res = {"overlap": [], "sequential": []}
for t in range(T):
    for name, f in (("overlap", fields[0]), ("sequential", fields[1])):
        flush.fill_(float(t))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        if name == "overlap":
            f.step(rp, rv, 0.35, check=False)
        else:
            for ph in (1, 2, 4):
                f.step_phase(ph, rp, rv, 0.35)
        e1.record(st)
        torch.cuda.synchronize()
        res[name].append(e0.elapsed_time(e1))
assert torch.equal(fields[0].pos_t, fields[1].pos_t) and torch.equal(fields[0].vel_t, fields[1].vel_t)
for k, v in res.items():
    print(f"{cfg} {k:10s} mean {np.mean(v):.4f} ms  median {np.median(v):.4f} ms")

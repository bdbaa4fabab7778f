"""The bench state of a config after W warm-up ticks, then ONE synchronous tick run
phase by phase (k_guide, k_astar, k_orca over all envs -- what bench.py's per-kernel
pass times), bracketed by cudaProfilerStart/Stop for
``ncu --profile-from-start off``.   python tools/tick_once.py cfg2 [W]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField  # noqa: E402
from paper_2505_00690_b200.rng import child_seeds_device  # noqa: E402
from paper_2505_00690_b200.urbangen import SceneSampler  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 20
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
run_seeds = child_seeds_device(env, "crowd-run").cpu().numpy().view(np.uint64)
f = CrowdField(b, CrowdConfig(neighbor_distance=C["nd"]), [int(x) for x in run_seeds])
f.set_from_spawn(b)
pick = (bench.robot_picks(E, 0).to(dev) * b.walk_n.double()).long()
cell = b.walk.gather(1, pick[:, None])[:, 0].long()
rp = torch.stack([((cell % nx).double() + 0.5) * C["res"], ((cell // nx).double() + 0.5) * C["res"]], 1)
rp = rp.contiguous()
rv = torch.zeros_like(rp)
for _ in range(W):
    f.step(rp, rv, 0.35, check=False)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
flush.fill_(1.0)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for ph in (1, 2, 4):
    f.step_phase(ph, rp, rv, 0.35)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
f.check_flags()
print(cfg, "tick", W, "stats", f.stats())

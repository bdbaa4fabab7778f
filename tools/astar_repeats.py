"""Count replanning requests that repeat the agent's previous (start, goal) exactly (GPU)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_2505_00690_b200 import _lib
from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
from paper_2505_00690_b200.rng import child_seeds_device
from paper_2505_00690_b200.urbangen import SceneSampler
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
CFG = bench.CFG
E = CFG["envs"]; dev = torch.device("cuda")
spec = bench.make_spec(); nx = int(np.ceil(CFG["extent"] / CFG["res"]))
zero = torch.zeros(E, dtype=torch.int64, device=dev)
es = child_seeds_device(zero, "env", torch.arange(E, device=dev))
sampler = SceneSampler(spec, E, device=dev)
sampler.sample(es, child_seeds_device(es, "crowd", 0), check=False)
b = sampler.batch
rs = child_seeds_device(es, "crowd-run").cpu().numpy().view(np.uint64)
f = CrowdField(b, CrowdConfig(neighbor_distance=CFG["nd"]), [int(s) for s in rs], device=dev)
f.set_from_spawn(b); f.prepare_step()
g = torch.Generator(device="cpu").manual_seed(1234)
pick = (torch.rand(E, generator=g).to(dev) * b.walk_n.double()).long()
cell = b.walk.gather(1, pick[:, None])[:, 0].long()
rpos = torch.stack([((cell % nx).double() + 0.5) * CFG["res"], ((cell // nx).double() + 0.5) * CFG["res"]], 1).contiguous()
rvel = torch.zeros_like(rpos)
last = {}
tot = rep = 0
tot_exp = rep_exp = 0
for k in range(steps):
    f.step_phase(1, rpos, rvel)
    n = int(f.flags_t[4].item())
    req = f.astar_req_t[:n].cpu().numpy()
    f.counters_t.zero_()
    dbg = torch.zeros((max(n, 1), 8), dtype=torch.int64, device=dev)
    f.step_phase(2, rpos, rvel)
    f.step_phase(4, rpos, rvel)
    for e_, a_, s_, g_ in req:
        key = (e_, a_)
        tot += 1
        if last.get(key) == (s_, g_):
            rep += 1
        last[key] = (s_, g_)
print(f"requests {tot} repeats {rep} ({100*rep/max(tot,1):.1f}%) over {steps} ticks")

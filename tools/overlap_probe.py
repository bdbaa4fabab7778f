"""Overlapped tick (cw_crowd_step) vs the three phases run back to back (GPU)."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
from paper_2505_00690_b200.rng import child_seeds_device
from paper_2505_00690_b200.urbangen import SceneSampler
CFG = bench.CFG
E = CFG["envs"]; dev = torch.device("cuda")
spec = bench.make_spec(); nx = int(np.ceil(CFG["extent"] / CFG["res"]))
es = child_seeds_device(torch.zeros(E, dtype=torch.int64, device=dev), "env", torch.arange(E, device=dev))
s = SceneSampler(spec, E, device=dev); s.sample(es, child_seeds_device(es, "crowd", 0), check=False)
b = s.batch
rs = child_seeds_device(es, "crowd-run").cpu().numpy().view(np.uint64)
f = CrowdField(b, CrowdConfig(neighbor_distance=CFG["nd"]), [int(x) for x in rs], device=dev)
f.set_from_spawn(b); f.prepare_step()
rpos = torch.full((E, 2), 16.0, dtype=torch.float64, device=dev); rvel = torch.zeros_like(rpos)
for _ in range(20):
    f.step(rpos, rvel, check=False)
st = torch.cuda.current_stream()
ev = lambda: torch.cuda.Event(enable_timing=True)
ov, seq = [], []
for k in range(40):
    a, c = ev(), ev()
    if k % 2 == 0:
        a.record(st); f.step(rpos, rvel, check=False); c.record(st)
        torch.cuda.synchronize(); ov.append(a.elapsed_time(c))
    else:
        a.record(st)
        for ph in (1, 2, 4):
            f.step_phase(ph, rpos, rvel)
        c.record(st)
        torch.cuda.synchronize(); seq.append(a.elapsed_time(c))
print(f"overlapped {np.mean(ov):.3f} ms   sequential {np.mean(seq):.3f} ms  (alternating ticks, no L2 flush)")

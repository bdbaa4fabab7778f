"""How often does a tick's A* request repeat the same (env, agent, start cell, goal
cell) as one of the previous ticks' requests, and how much of the tick's longest
search is such a repeat?  (cfg2 bench setup, synchronous ticks.)"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2505_00690_b200 import _lib  # noqa: E402
from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField  # noqa: E402
from paper_2505_00690_b200.rng import child_seeds_device  # noqa: E402
from paper_2505_00690_b200.urbangen import SceneSampler  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfgname = sys.argv[3] if len(sys.argv) > 3 else "cfg2"
bench.CFG.clear()
bench.CFG.update(bench.CONFIGS[cfgname])
CFG = bench.CFG
E = CFG["envs"]
dev = torch.device("cuda")
nx = int(np.ceil(CFG["extent"] / CFG["res"]))
zero = torch.zeros(E, dtype=torch.int64, device=dev)
env_seeds = child_seeds_device(zero, "env", torch.arange(E, device=dev))
sampler = SceneSampler(bench.make_spec(), E, device=dev)
b = sampler.sample(env_seeds, child_seeds_device(env_seeds, "crowd", 0))
run_seeds = child_seeds_device(env_seeds, "crowd-run").cpu().numpy().view(np.uint64)
f = CrowdField(b, CrowdConfig(neighbor_distance=CFG["nd"]), [int(s) for s in run_seeds])
f.set_from_spawn(b)
f.prepare_step()
pick = (bench.robot_picks(E, 0).to(dev) * b.walk_n.double()).long()
cell = b.walk.gather(1, pick[:, None])[:, 0].long()
rpos = torch.stack([((cell % nx).double() + 0.5) * CFG["res"], ((cell // nx).double() + 0.5) * CFG["res"]], 1)
rpos = rpos.contiguous()
rvel = torch.zeros_like(rpos)
for _ in range(warm):
    f.step(rpos, rvel, 0.35, check=False)
torch.cuda.synchronize()
L = _lib.lib()


def run(ph):
    _lib.check(L.cw_crowd_step_phases(f._p, f._s, _lib.ptr(rpos), _lib.ptr(rvel), 0.35, None, f._step_nt(), ph,
                                      None), "phase")


seen = {}   # (env, agent) -> set of (start, goal) searched before
tot = rep_n = 0
rep_cyc = tot_cyc = 0.0
max_is_rep = 0
last = {}
for k in range(steps):
    run(1)
    torch.cuda.synchronize()
    nreq = int(f.flags_t[4].item())
    req = f.astar_req_t[:nreq].cpu().numpy().copy()
    dbg = torch.zeros((max(nreq, 1), 8), dtype=torch.int64, device=dev)
    f.counters_t[14] = dbg.data_ptr()
    run(2)
    torch.cuda.synchronize()
    f.counters_t[14] = 0
    d = dbg.cpu().numpy()[:nreq]
    run(4)
    torch.cuda.synchronize()
    reps = np.array([(int(r[2]), int(r[3])) in seen.get((int(r[0]), int(r[1])), ()) for r in req], bool)
    prev = np.array([last.get((int(r[0]), int(r[1]))) == (int(r[2]), int(r[3])) for r in req], bool)
    tot += nreq
    rep_n += int(reps.sum())
    tot_cyc += float(d[:, 0].sum())
    rep_cyc += float(d[reps, 0].sum())
    if nreq:
        im = int(np.argmax(d[:, 0]))
        max_is_rep += int(reps[im])
        print(f"tick {k}: req {nreq} repeats {int(reps.sum())} (prev tick {int(prev.sum())}); longest "
              f"{d[im, 0] / 1e6:.2f}M cyc exp {d[im, 1]} repeat={bool(reps[im])} env {req[im, 0]} agent {req[im, 1]}",
              flush=True)
    for r in req:
        seen.setdefault((int(r[0]), int(r[1])), set()).add((int(r[2]), int(r[3])))
        last[(int(r[0]), int(r[1]))] = (int(r[2]), int(r[3]))
print(f"requests {tot}, repeats {rep_n} ({rep_n / max(tot, 1):.1%}), repeat cycles {rep_cyc / max(tot_cyc, 1):.1%}, "
      f"ticks whose longest search is a repeat: {max_is_rep}/{steps}")

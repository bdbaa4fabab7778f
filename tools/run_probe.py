"""Synchronous ticks vs cw_crowd_run on a bench config (GPU).

Usage: python tools/run_probe.py [ticks] [config]
Prints ms per tick for: T x CrowdField.step (no L2 flush), CrowdField.run(T),
and checks the two leave identical states.
"""
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

T = int(sys.argv[1]) if len(sys.argv) > 1 else 100
cfgname = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
bench.CFG.clear()
bench.CFG.update(bench.CONFIGS[cfgname])
CFG = bench.CFG
E = int(os.environ.get("PROBE_ENVS", CFG["envs"]))
dev = torch.device("cuda")
_lib.build()
spec = bench.make_spec()
nx = int(np.ceil(CFG["extent"] / CFG["res"]))
zero = torch.zeros(E, dtype=torch.int64, device=dev)
env_seeds = child_seeds_device(zero, "env", torch.arange(E, device=dev))
crowd_seeds = child_seeds_device(env_seeds, "crowd", 0)
run_seeds = [int(s) for s in child_seeds_device(env_seeds, "crowd-run").cpu().numpy().view(np.uint64)]
sampler = SceneSampler(spec, E, device=dev)
b = sampler.sample(env_seeds, crowd_seeds, check=False)
g = torch.Generator(device="cpu").manual_seed(1234)
pick = (torch.rand(E, generator=g).to(dev) * b.walk_n.double()).long()
cell = b.walk.gather(1, pick[:, None])[:, 0].long()
rpos = torch.stack([((cell % nx).double() + 0.5) * CFG["res"],
                    ((cell // nx).double() + 0.5) * CFG["res"]], dim=1).contiguous()
rvel = torch.zeros_like(rpos)
fields = []
for _ in range(2):
    f = CrowdField(b, CrowdConfig(neighbor_distance=CFG["nd"]), run_seeds, device=dev,
                   astar_warps=int(os.environ["PROBE_ASTAR_WARPS"]) if "PROBE_ASTAR_WARPS" in os.environ else None,
                   threads=int(os.environ.get("PROBE_THREADS", 128)))
    f.run_threads = int(os.environ["PROBE_RUN_THREADS"]) if "PROBE_RUN_THREADS" in os.environ else None
    f.set_from_spawn(b)
    f.prepare_step()
    for _ in range(20):
        f.step(rpos, rvel, 0.35, check=False)
    fields.append(f)
torch.cuda.synchronize()
f, h = fields
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(T):
    f.step(rpos, rvel, 0.35, check=False)
e1.record(st)
torch.cuda.synchronize()
sync_ms = e0.elapsed_time(e1) / T
h.run(1, rpos, rvel, 0.35)   # warm the run path (first-call attributes)
torch.cuda.synchronize()
f.step(rpos, rvel, 0.35, check=False)
h.counters_t.zero_()
e0.record(st)
h.run(T, rpos, rvel, 0.35)
e1.record(st)
torch.cuda.synchronize()
run_ms = e0.elapsed_time(e1) / T
same = True
for k in ("pos_t", "vel_t", "goal_t", "waypoint_t", "path_n_t", "last_gap_t"):
    x, y = getattr(f, k).cpu().numpy(), getattr(h, k).cpu().numpy()
    if not np.array_equal(x, y):
        same = False
        bad = np.argwhere(x != y)
        envs = np.unique(bad[:, 0]) if bad.ndim > 1 and bad.shape[1] > 0 else bad
        print(f"  MISMATCH {k}: {len(bad)} entries, envs {envs[:10]} (of {len(envs)})")
print("  flags sync", f.flags_t.cpu().numpy()[:2], "run", h.flags_t.cpu().numpy()[:2])
c = h.counters_t.cpu().numpy()
clk = 1.92e6   # cycles per ms (approx. boost clock)
print(f"  run: expansions {c[0]:,} search warp-cycles {c[4]/1e6:.0f}M (= {c[4]/clk/T:.2f} warp-ms/tick), "
      f"max search {c[5]/1e6:.1f}M cyc, orca CTA-cycles {c[6]/1e6:.0f}M (= {c[6]/clk/T:.2f} CTA-ms/tick), "
      f"guide CTA-cycles {c[8]/1e6:.0f}M (= {c[8]/clk/T:.2f} CTA-ms/tick)")
print(f"{cfgname} E={E} T={T}: sync {sync_ms:.3f} ms/tick ({E / sync_ms * 1e3:,.0f} env-steps/s); "
      f"run {run_ms:.3f} ms/tick ({E / run_ms * 1e3:,.0f} env-steps/s); identical={same}")

"""Per-tick CrowdField.step time with and without the next-tick A* prefetch, and the
prefetch counters (hits / waits on a running prediction / claims of a queued one)
against the tick's real replan count.   python tools/prefetch_probe.py [config] [ticks]"""
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
T = int(sys.argv[2]) if len(sys.argv) > 2 else 40
bench.CFG.clear()
bench.CFG.update(bench.CONFIGS[cfg])
E = int(os.environ.get("LAB_ENVS", bench.CFG["envs"]))
dev = torch.device("cuda")
zero = torch.zeros(E, dtype=torch.int64, device=dev)
env = child_seeds_device(zero, "env", torch.arange(E, device=dev))
s = SceneSampler(bench.make_spec(), E)
s.sample(env, child_seeds_device(env, "crowd", 0))
b = s.batch
seeds = [int(x) for x in child_seeds_device(env, "crowd-run").cpu().numpy().view(np.uint64)]
nx = b.labels.shape[2]
res = float(b.params.res)
g = torch.Generator(device="cpu").manual_seed(1234)
pick = (torch.rand(E, generator=g).to(dev) * b.walk_n.double()).long()
cell = b.walk.gather(1, pick[:, None])[:, 0].long()
rp = torch.stack([((cell % nx).double() + 0.5) * res, ((cell // nx).double() + 0.5) * res], 1).contiguous()
rv = torch.zeros_like(rp)
st = torch.cuda.current_stream()
for pf in (True, False):
    f = CrowdField(b, CrowdConfig(neighbor_distance=bench.CFG["nd"]), seeds, prefetch=pf)
    f.set_from_spawn(b)
    for _ in range(20):
        f.step(rp, rv, 0.35, check=False)
    torch.cuda.synchronize()
    p0 = f.prefetch_stats()
    ts, reqs = [], []
    for k in range(T):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        f.step(rp, rv, 0.35, check=False)
        e1.record(st)
        st.synchronize()   # the caller's stream only: the prefetch keeps running
        ts.append(e0.elapsed_time(e1))
        reqs.append(int(f.flags_t[4].item()))
    p1 = f.prefetch_stats()
    d = {k: p1[k] - p0[k] for k in p1} if pf else {}
    print(f"prefetch={pf}: {np.mean(ts):.3f} ms/tick (median {np.median(ts):.3f}, max {np.max(ts):.3f}); "
          f"replans {sum(reqs)} ({np.mean(reqs):.1f}/tick) {d}", flush=True)
    f._spec_free()

import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import bench
from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
from paper_2505_00690_b200.rng import child_seeds_device
from paper_2505_00690_b200.urbangen import SceneSampler
bench.CFG.clear(); bench.CFG.update(bench.CONFIGS["cfg5"])
E = bench.CFG["envs"]; dev = torch.device("cuda")
zero = torch.zeros(E, dtype=torch.int64, device=dev)
env = child_seeds_device(zero, "env", torch.arange(E, device=dev))
s = SceneSampler(bench.make_spec(), E); s.sample(env, child_seeds_device(env, "crowd", 0))
seeds = [int(x) for x in child_seeds_device(env, "crowd-run").cpu().numpy().view(np.uint64)]
f = CrowdField(s.batch, CrowdConfig(neighbor_distance=bench.CFG["nd"]), seeds, prefetch=False)
f.set_from_spawn(s.batch)
for _ in range(20): f.step()
rng = np.random.default_rng(0); counts = torch.zeros(E, dtype=torch.int64, device=dev)
st = torch.cuda.current_stream()
for k in range(6):
    rows = np.flatnonzero(rng.random(E) < 0.02)
    sl = torch.from_numpy(rows).to(dev); counts[sl] += 1
    if k % 2 == 0:
        s.sample(child_seeds_device(env[sl], "resample", counts[sl]), child_seeds_device(env[sl], "crowd", counts[sl]), slots=sl)
        f.set_from_spawn(s.batch, rows=sl)
    torch.cuda.synchronize()
    for ph in (1, 2, 4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f.counters_t.zero_()
        e0.record(st); f.step_phase(ph); e1.record(st); torch.cuda.synchronize()
        if ph == 2:
            req = int(f.flags_t[4].item()); c = f.counters_t.cpu().numpy()
            print(f"tick {k} resampled={k%2==0} rows={len(rows)} requests={req} exp={c[0]} astar_ms={e0.elapsed_time(e1):.2f} max_cyc={c[5]/1e6:.1f}M")

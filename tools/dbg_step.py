import sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
from paper_2505_00690_b200.rng import child_seeds_device
from paper_2505_00690_b200.urbangen import SceneSampler
E = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
spec = bench.make_spec()
dev = torch.device('cuda')
zero = torch.zeros(E, dtype=torch.int64, device=dev)
es = child_seeds_device(zero, 'env', torch.arange(E, device=dev))
cs = child_seeds_device(es, 'crowd', 0)
rs = child_seeds_device(es, 'crowd-run').cpu().numpy().view(np.uint64)
b = SceneSampler(spec, E).sample(es, cs)
f = CrowdField(b, CrowdConfig(), [int(s) for s in rs])
f.set_from_spawn(b)
f.prepare_step()
for t in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    f.counters_t.zero_()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    f.step(check=False)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    st = f.stats()
    ex = max(1, st["astar_expansions"]); print(t, f"{dt*1e3:.2f} ms", "exp", st["astar_expansions"], "cyc/exp", round(st["astar_cycles"]/ex), "max search ms", round(st["astar_max_cycles"]/1.9e6, 2), "orca cta max ms", round(st["cta_max_cycles"]/1.9e6, 3))

"""Run the cfg2 sampling pipeline a few times (for ncu launch lists / timing)."""
import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
from paper_2505_00690_b200.rng import child_seeds_device
from paper_2505_00690_b200.urbangen import SceneSampler
E = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = bench.make_spec()
dev = torch.device('cuda')
zero = torch.zeros(E, dtype=torch.int64, device=dev)
es = child_seeds_device(zero, 'env', torch.arange(E, device=dev))
cs = child_seeds_device(es, 'crowd', 0)
s = SceneSampler(spec, E)
for r in range(reps):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s.sample(es, cs, check=False)
    torch.cuda.synchronize(); print(f"rep {r}: {1e3*(time.perf_counter()-t0):.2f} ms")
s.batch.check_status()

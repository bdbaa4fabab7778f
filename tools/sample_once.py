"""One sampling batch of a bench config (for ncu captures of the sampling kernels)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_00690_b200.rng import child_seeds_device  # noqa: E402
from paper_2505_00690_b200.urbangen import SceneSampler  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
bench.CFG.clear()
bench.CFG.update(bench.CONFIGS[cfg])
E = bench.CFG["envs"] if len(sys.argv) < 3 else int(sys.argv[2])
zero = torch.zeros(E, dtype=torch.int64, device="cuda")
es = child_seeds_device(zero, "env", torch.arange(E, device="cuda"))
s = SceneSampler(bench.make_spec(), E)
s.sample(es, child_seeds_device(es, "crowd", 0))
torch.cuda.synchronize()
print("sampled", E)

"""Locate the first tick where CrowdField.run diverges from synchronous steps (GPU).
Usage: python tools/run_diff.py [ticks] [config]"""
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
cfgname = sys.argv[2] if len(sys.argv) > 2 else "cfg5"
bench.CFG.clear()
bench.CFG.update(bench.CONFIGS[cfgname])
CFG = bench.CFG
E = int(os.environ.get("PROBE_ENVS", 1024))
dev = torch.device("cuda")
_lib.build()
spec = bench.make_spec()
nx = int(np.ceil(CFG["extent"] / CFG["res"]))
zero = torch.zeros(E, dtype=torch.int64, device=dev)
env_seeds = child_seeds_device(zero, "env", torch.arange(E, device=dev))
crowd_seeds = child_seeds_device(env_seeds, "crowd", 0)
run_seeds = [int(s) for s in child_seeds_device(env_seeds, "crowd-run").cpu().numpy().view(np.uint64)]
b = SceneSampler(spec, E, device=dev).sample(env_seeds, crowd_seeds, check=False)
g = torch.Generator(device="cpu").manual_seed(1234)
pick = (torch.rand(E, generator=g).to(dev) * b.walk_n.double()).long()
cell = b.walk.gather(1, pick[:, None])[:, 0].long()
rpos = torch.stack([((cell % nx).double() + 0.5) * CFG["res"],
                    ((cell // nx).double() + 0.5) * CFG["res"]], dim=1).contiguous()
rvel = torch.zeros_like(rpos)
fs = []
for _ in range(2):
    f = CrowdField(b, CrowdConfig(neighbor_distance=CFG["nd"]), run_seeds, device=dev)
    f.set_from_spawn(b)
    f.prepare_step()
    fs.append(f)
f, h = fs
keys = ("pos_t", "vel_t", "goal_t", "waypoint_t", "path_head_t", "path_n_t", "path_cells_t")
mode = os.environ.get("DIFF_MODE", "run1")
K = int(os.environ.get("DIFF_CHUNK", 1))
for t in range(0, T, K):
    for _ in range(K):
        f.step(rpos, rvel, 0.35, check=False)
    if mode == "run1":
        h.run(K, rpos, rvel, 0.35)
    else:
        for _ in range(K):
            h.step(rpos, rvel, 0.35, check=False)
    torch.cuda.synchronize()
    for k in keys:
        x, y = getattr(f, k).cpu().numpy(), getattr(h, k).cpu().numpy()
        if not np.array_equal(x, y):
            idx = np.unique(np.argwhere(x != y)[:, :2], axis=0)
            print(f"tick {t}: {k} differs at (env, agent) {idx[:6].tolist()}")
            for e, a in idx[:2]:
                print("   sync: head", int(f.path_head_t[e, a]), "n", int(f.path_n_t[e, a]),
                      "wp", f.waypoint_t[e, a].tolist(), "pos", f.pos_t[e, a].tolist(), "goal", f.goal_t[e, a].tolist())
                print("   run : head", int(h.path_head_t[e, a]), "n", int(h.path_n_t[e, a]),
                      "wp", h.waypoint_t[e, a].tolist(), "pos", h.pos_t[e, a].tolist(), "goal", h.goal_t[e, a].tolist())
            sys.exit(0)
print(f"{mode}: identical over {T} ticks")

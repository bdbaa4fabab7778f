"""Check device A* results of chosen envs against the oracle A*, tick by tick (GPU).
Usage: python tools/astar_check.py [ticks] [config] [env,env,...]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import crowd as C  # noqa: E402
from paper_2505_00690_b200 import _lib  # noqa: E402
from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField  # noqa: E402
from paper_2505_00690_b200.rng import child_seeds_device  # noqa: E402
from paper_2505_00690_b200.urbangen import SceneSampler  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 100
cfgname = sys.argv[2] if len(sys.argv) > 2 else "cfg5"
watch = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [360]
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
f = CrowdField(b, CrowdConfig(neighbor_distance=CFG["nd"]), run_seeds, device=dev)
f.set_from_spawn(b)
f.prepare_step()
if os.environ.get("CHECK_W"):
    f._p.astar_warps = int(os.environ["CHECK_W"])
L = _lib.lib()
labs = {e: b.labels[e].cpu().numpy() != 0 for e in watch}


def phase(ph):
    _lib.check(L.cw_crowd_step_phases(f._p, f._s, _lib.ptr(rpos), _lib.ptr(rvel), 0.35, None, f._step_nt(), ph,
                                      _lib.stream_ptr(None)), "phase")


checked = bad = 0
for t in range(T):
    phase(1)
    torch.cuda.synchronize()
    nreq = int(f.flags_t[4])
    reqs = f.astar_req_t[:nreq].cpu().numpy()
    phase(2)
    torch.cuda.synchronize()
    per_tick = 0
    cap = int(os.environ.get("ASTAR_CHECK_MAX", 1 << 30))
    for e, a, st, gl in reqs:
        if e not in labs or per_tick >= cap:
            continue
        per_tick += 1
        ref = C.astar(labs[e], (st // nx, st % nx), (gl // nx, gl % nx))
        n = int(f.path_n_t[e, a])
        hd = int(f.path_head_t[e, a])
        cells = f.path_cells_t[e, a, hd:hd + max(n - 1, 0)].cpu().numpy()
        want = [] if ref is None else [r * nx + c for r, c in ref[1:]]
        ok = (ref is None and n == 1) or (ref is not None and n == len(ref) and list(cells) == want)
        checked += 1
        if not ok:
            bad += 1
            print(f"tick {t} env {e} agent {a} start {divmod(int(st), nx)} goal {divmod(int(gl), nx)}: "
                  f"device n {n} oracle n {None if ref is None else len(ref)}", flush=True)
            np.savez(os.path.join(ROOT, "gpurun_out", f"astar_bad_{t}_{e}_{a}.npz"), labels=labs[e],
                     start=st, goal=gl, dev_cells=cells, dev_n=n)
    phase(4)
print(f"checked {checked} searches of envs {watch}: {bad} wrong")

"""Find A* requests whose device result depends on the search shape (GPU).

Steps a bench config; every tick runs k_guide, then the tick's queued searches
twice -- latency shape (1 warp, NC 1024) and throughput shape (4 warps, NC 512)
-- from the same pre-search state, compares path_cells / path_n / waypoint,
and checks any mismatch against the oracle A* (oracle/crowd.py astar).
Usage: python tools/astar_diff.py [ticks] [config]
"""
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

T = int(sys.argv[1]) if len(sys.argv) > 1 else 60
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
f = CrowdField(b, CrowdConfig(neighbor_distance=CFG["nd"]), run_seeds, device=dev)
f.set_from_spawn(b)
f.prepare_step()
L = _lib.lib()


def phase(ph):
    _lib.check(L.cw_crowd_step_phases(f._p, f._s, _lib.ptr(rpos), _lib.ptr(rvel), 0.35, None, f._step_nt(), ph,
                                      _lib.stream_ptr(None)), "phase")


names = ("path_cells_t", "path_head_t", "path_n_t", "waypoint_t")
bad = 0
for t in range(T):
    phase(1)
    torch.cuda.synchronize()
    nreq = int(f.flags_t[4])
    snap = {k: getattr(f, k).clone() for k in names}
    out = {}
    for w in (1, 4):
        for k in names:
            getattr(f, k).copy_(snap[k])
        f.flags_t[5] = 0
        f._p.astar_warps = w
        phase(2)
        torch.cuda.synchronize()
        out[w] = {k: getattr(f, k).clone() for k in names}
    reqs = f.astar_req_t[:nreq].cpu().numpy()
    for k in names:
        x, y = out[1][k].cpu().numpy(), out[4][k].cpu().numpy()
        if not np.array_equal(x, y):
            idx = np.unique(np.argwhere(x != y)[:, :2], axis=0)
            for e, a in idx[:4]:
                r = [q for q in reqs if q[0] == e and q[1] == a]
                lab = b.labels[e].cpu().numpy()
                line = f"tick {t} field {k} env {e} agent {a} req {r}"
                if r:
                    st, gl = int(r[0][2]), int(r[0][3])
                    ref = C.astar(lab != 0, (st // nx, st % nx), (gl // nx, gl % nx))
                    n1, n4 = int(out[1]["path_n_t"][e, a]), int(out[4]["path_n_t"][e, a])
                    line += f" oracle len {None if ref is None else len(ref)} W1 path_n {n1} W4 path_n {n4}"
                print(line, flush=True)
                bad += 1
            break
    phase(4)
print(f"{T} ticks, {bad} mismatching searches")

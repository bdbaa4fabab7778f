"""Lab for the A* kernel on live cfg2 replanning queues (GPU).

Runs the bench setup, then for each measured tick: k_guide, the timed
k_astar with per-search debug records (counters[14] -> buffer), k_orca.
Usage: python tools/astar_lab.py [steps] [warmup] [unused] [config]
"""
import ctypes
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

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfgname = sys.argv[4] if len(sys.argv) > 4 else "cfg2"
bench.CFG.clear()
bench.CFG.update(bench.CONFIGS[cfgname])
CFG = bench.CFG
E = int(os.environ.get("LAB_ENVS", CFG["envs"]))
dev = torch.device("cuda")
_lib.build()
spec = bench.make_spec()
nx = int(np.ceil(CFG["extent"] / CFG["res"]))
zero = torch.zeros(E, dtype=torch.int64, device=dev)
env_seeds = child_seeds_device(zero, "env", torch.arange(E, device=dev))
crowd_seeds = child_seeds_device(env_seeds, "crowd", 0)
run_seeds = child_seeds_device(env_seeds, "crowd-run").cpu().numpy().view(np.uint64)
sampler = SceneSampler(spec, E, device=dev)
sampler.sample(env_seeds, crowd_seeds, check=False)
b = sampler.batch
f = CrowdField(b, CrowdConfig(neighbor_distance=CFG["nd"]), [int(s) for s in run_seeds], device=dev)
f.set_from_spawn(b)
f.prepare_step()
g = torch.Generator(device="cpu").manual_seed(1234)
pick = (torch.rand(E, generator=g).to(dev) * b.walk_n.double()).long()
cell = b.walk.gather(1, pick[:, None])[:, 0].long()
rpos = torch.stack([((cell % nx).double() + 0.5) * CFG["res"],
                    ((cell // nx).double() + 0.5) * CFG["res"]], dim=1).contiguous()
rvel = torch.zeros_like(rpos)
for _ in range(warm):
    f.step(rpos, rvel, 0.35, check=False)
torch.cuda.synchronize()
f.check_flags()

L = _lib.lib()
st = torch.cuda.current_stream()


def run(phases):
    err = L.cw_crowd_step_phases(f._p, f._s, _lib.ptr(rpos), _lib.ptr(rvel), 0.35, None, f._step_nt(),
                                 phases, _lib.stream_ptr(None))
    _lib.check(err, "phase")


tot = 0.0
tick_max = []
mats = []
for k in range(steps):
    run(1)
    torch.cuda.synchronize()
    nreq = int(f.flags_t[4].item())
    f.counters_t.zero_()
    dbg = torch.zeros((max(nreq, 1), 8), dtype=torch.int64, device=dev)
    f.counters_t[14] = dbg.data_ptr()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    run(2)
    e1.record(st)
    torch.cuda.synchronize()
    f.counters_t[14] = 0
    t = e0.elapsed_time(e1)
    c = f.counters_t.cpu().numpy().copy()
    d = dbg.cpu().numpy()
    if os.environ.get("LAB_ENVSUM"):
        per_env = np.zeros(E)
        np.maximum.at(per_env, d[:nreq, 2].astype(np.int64), d[:nreq, 0].astype(np.float64))
        env_sum = per_env if k == 0 else env_sum + per_env
        tick_max.append(per_env.max())
        mats.append(per_env.copy())
        if k == 0:
            env_cnt = np.zeros(E); env_exp = np.zeros(E); env_ticks = np.zeros(E)
        np.add.at(env_cnt, d[:nreq, 2].astype(np.int64), 1)
        np.add.at(env_exp, d[:nreq, 2].astype(np.int64), d[:nreq, 1].astype(np.float64))
        env_ticks[np.unique(d[:nreq, 2].astype(np.int64))] += 1
    for r_ in d[np.argsort(-d[:, 0])[:2]]:
        if os.environ.get("LAB_PHASES"):   # build with -DCW_ASTAR_PHASES
            x_ = max(r_[1], 1)
            print(f"      per exp: head inserts {r_[4]/x_:5.2f} insert cyc {r_[5]/x_:6.0f} "
                  f"held {r_[6]/x_:5.2f} refill cyc {r_[7]/x_:6.0f}")
        print(f"   search cyc {r_[0]/1e6:6.2f}M exp {r_[1]:6d} cyc/exp {r_[0]/max(r_[1],1):6.0f} env {r_[2]:6d} "
              f"tiles {r_[3]:6d}")
    if os.environ.get("LAB_PHASES"):
        a_ = d[:nreq].sum(axis=0).astype(np.float64)
        x_ = max(a_[1], 1)
        print(f"   all: cyc/exp {a_[0]/x_:6.0f} inserts {a_[4]/x_:5.2f} insert cyc {a_[5]/x_:6.0f} "
              f"held {a_[6]/x_:5.2f} refill cyc {a_[7]/x_:6.0f}")
    f.check_flags()
    run(4)
    tot += t
    print(f"step {k:3d} req {nreq:5d} exp {c[0]:8d} glob {c[10]:3d} max_cyc {c[5]/1e6:7.2f}M  ms {t:7.3f}", flush=True)
print(f"TOTAL {tot:.2f} ms over {steps} ticks")
if os.environ.get("LAB_ENVSUM"):
    srt = np.sort(env_sum)[::-1]
    M = np.stack(mats)   # (ticks, E)
    np.save(os.path.join(ROOT, "gpurun_out", "lab_env_tick.npy"), M)
    for G in (1, 2, 4, 8, 16, 32, 64, 128):
        grp = M.reshape(M.shape[0], G, -1).max(axis=2).sum(axis=0)
        print(f"  G={G:4d}: max over groups of summed tick-max {grp.max()/1e6:7.1f}M cycles")
    top = np.argsort(-env_sum)[:6]
    for e_ in top:
        print(f"  env {e_}: summed cycles {env_sum[e_]/1e6:.1f}M, searches {env_cnt[e_]:.0f} in {env_ticks[e_]:.0f} "
              f"ticks, expansions {env_exp[e_]:.0f} ({env_exp[e_]/max(env_cnt[e_],1):.0f}/search)")
    print(f"sum over ticks of max-search cycles {sum(tick_max)/1e6:.1f}M; max over envs of summed "
          f"cycles {srt[0]/1e6:.1f}M; next envs {[round(v/1e6, 1) for v in srt[1:8]]}")


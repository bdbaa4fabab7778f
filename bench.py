"""Benchmark: async scene sampling + crowd dynamics step on B200 (BASELINE.json configs[1]).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--envs E]

Workload (cfg2): E=1024 envs per GPU, 32 m x 32 m at 0.125 m (256x256 grid),
64 objects, 32 pedestrians per env, NavDynamic, terrain mix 0.25 each, dt 0.05,
seeds child_seed(0, "env", global_env_id).  A "step" is one CrowdField.step over
every env of the rank (one cw_crowd_step launch).  Scenes/s is the whole
cw_sample_scenes pipeline over the same E envs.  Under torchrun each rank owns
E envs (weak scaling, no data-path collective; one NCCL all_gather of per-env
stats at the end).  ``--impl reference`` times the reference's CPU algorithm
(the oracle port, all host cores) on a bounded sample of the same workload.
"""

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MIX = {"Flat": 0.25, "Slope": 0.25, "Stair": 0.25, "Rough": 0.25}
# BASELINE.json configs mapped onto the reference API.  cfg2 is the
# bench default (the metric's single-GPU config); the others are --config runs.
CONFIGS = {
    "cfg1": dict(envs=16, extent=32.0, res=0.125 * 2, objects=20, peds=8, task="NavDynamic", nd=5.0,
                 resample=0.0, steps_cfg=100),
    "cfg2": dict(envs=1024, extent=32.0, res=0.125, objects=64, peds=32, task="NavDynamic", nd=5.0,
                 resample=0.0, steps_cfg=500),
    "cfg3": dict(envs=4096, extent=32.0, res=0.125, objects=100, peds=64, task="NavDynamic", nd=5.0,
                 resample=0.0, steps_cfg=1000),
    "cfg4": dict(envs=512, extent=64.0, res=0.125, objects=0, peds=1024, task="NavClear", nd=3.0,
                 resample=0.0, steps_cfg=200),
    "cfg5": dict(envs=8192, extent=32.0, res=0.125, objects=128, peds=48, task="NavDynamic", nd=5.0,
                 resample=0.02, steps_cfg=2000),
}
CFG = dict(CONFIGS["cfg2"])
METRIC = "env-steps/sec and scenes sampled/sec at N envs on 1/2/4/8 B200; % of HBM peak"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def traffic_of(kernel):
    """dram read+write bytes per launch of `kernel` from the committed ncu --set full
    capture (profiles/r1_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1_traffic.json")) as fh:
            k = json.load(fh)["kernels"][kernel]
        return float(k["dram_read_bytes"] + k["dram_write_bytes"])
    except Exception:
        return None


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None
        self.path = f"/tmp/cw_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [l.split(",") for l in open(self.path).read().strip().splitlines()]
            rows = [[c.strip() for c in r] for r in rows if len(r) >= 7]
            sm = [float(r[0]) for r in rows]
            mx = max(float(r[1]) for r in rows)
            reasons = set()
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for r in rows:
                for n, v in zip(names, r[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                    "samples": len(rows)}
        except Exception as exc:  # no nvidia-smi
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": str(exc)[:80]}


def make_spec(cfg=None):
    from paper_2505_00690_b200.urbangen import SceneSpec, TaskKind
    cfg = cfg or CFG
    n = int(np.ceil(cfg["extent"] / cfg["res"]))
    base = int(np.floor(4.0 * (n * n * cfg["res"] * cfg["res"]) / 100.0 + 0.5))  # 41 at 32 m
    dens = cfg["objects"] / base if cfg["objects"] else 0.0
    return SceneSpec(seed=0, extent_m=(cfg["extent"], cfg["extent"]), task_kind=TaskKind(cfg["task"]),
                     object_density=dens, pedestrian_count=cfg["peds"],
                     terrain_mix=MIX, grid_resolution_m=cfg["res"])


# ============================================================================ ours
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2505_00690_b200 import _lib
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
    from paper_2505_00690_b200.rng import child_seeds_device
    from paper_2505_00690_b200.urbangen import SceneSampler

    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    _lib.build()
    from paper_2505_00690_b200 import shard
    E = args.envs
    spec = make_spec()
    nx = int(np.ceil(CFG["extent"] / CFG["res"]))
    zero = torch.zeros(E, dtype=torch.int64, device=dev)
    gids = torch.from_numpy(shard.env_ids(rank, world, E)).to(dev)   # rank owns [r*E, (r+1)*E)
    env_seeds = child_seeds_device(zero, "env", gids)
    crowd_seeds = child_seeds_device(env_seeds, "crowd", 0)
    run_seeds = child_seeds_device(env_seeds, "crowd-run").cpu().numpy().view(np.uint64)
    sampler = SceneSampler(spec, E, device=dev)

    # ---- scene sampling throughput (whole pipeline, E envs per launch sequence)
    st = torch.cuda.current_stream()
    for _ in range(max(1, args.sample_warmup)):
        sampler.sample(env_seeds, crowd_seeds, check=False)
    torch.cuda.synchronize()
    sampler.batch.check_status()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = args.sample_reps
    ev0.record(st)
    for _ in range(reps):
        sampler.sample(env_seeds, crowd_seeds, check=False)
    ev1.record(st)
    torch.cuda.synchronize()
    sample_ms = ev0.elapsed_time(ev1) / reps
    b = sampler.batch
    b.check_status()

    # ---- crowd
    f = CrowdField(b, CrowdConfig(neighbor_distance=CFG["nd"]), [int(s) for s in run_seeds], device=dev,
                   threads=args.threads)
    f.set_from_spawn(b)
    f.prepare_step()
    # robot: static at a seeded walkable cell per env (route anchors are §8f), zero velocity
    g = torch.Generator(device="cpu").manual_seed(1234 + rank)
    pick = (torch.rand(E, generator=g).to(dev) * b.walk_n.double()).long()
    cell = b.walk.gather(1, pick[:, None])[:, 0].long()
    rpos = torch.stack([((cell % nx).double() + 0.5) * CFG["res"],
                        ((cell // nx).double() + 0.5) * CFG["res"]], dim=1).contiguous()
    rvel = torch.zeros_like(rpos)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > L2
    for _ in range(args.warmup):
        f.step(rpos, rvel, 0.35, check=False)
    torch.cuda.synchronize()
    f.check_flags()
    f.counters_t.zero_()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    active = int(f.active_t.sum().item())
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    resampled = 0
    if CFG["resample"] > 0:
        # cfg5 driver: env i re-sampled at step t iff
        # make_rng(0, "resample-mix", t).random(E) < p, via BatchedEnv.reset semantics
        from paper_2505_00690_b200.rng import child_seed as _cs
        masks = [np.flatnonzero(np.random.Generator(np.random.PCG64(_cs(0, "resample-mix", k)))
                                .random(E * world)[rank * E:(rank + 1) * E] < CFG["resample"])
                 for k in range(args.steps)]
        counts = torch.zeros(E, dtype=torch.int64, device=dev)
    def resample_mix(k):
        nonlocal resampled
        if CFG["resample"] > 0 and masks[k].size:
            sl = torch.from_numpy(masks[k]).to(dev)
            counts[sl] += 1
            env_k = env_seeds[sl]
            new_scene = child_seeds_device(env_k, "resample", counts[sl])
            sampler.sample(new_scene, child_seeds_device(env_k, "crowd", counts[sl]), slots=sl,
                           check=False)
            f.set_from_spawn(b, rows=sl)
            resampled += int(masks[k].size)

    with Clocks(dev.index) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))          # L2 flush between timed steps (untimed)
            starts[k].record(st)
            resample_mix(k)
            mids[k].record(st)
            f.step(rpos, rvel, 0.35, check=False)
            ends[k].record(st)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f.check_flags()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    resample_ms = float(np.mean([s.elapsed_time(m) for s, m in zip(starts, mids)]))
    t_ms = float(sum(step_ms))
    counters = f.stats()
    # ---- per-kernel pass (same stream, events between the three launches)
    n_ph = min(args.steps, args.phase_steps)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n_ph)]
    f.counters_t.zero_()
    torch.cuda.synchronize()
    for k in range(n_ph):
        flush.fill_(float(k))
        ev[k][0].record(st)
        f.step_phase(1, rpos, rvel, 0.35)
        ev[k][1].record(st)
        f.step_phase(2, rpos, rvel, 0.35)
        ev[k][2].record(st)
        f.step_phase(4, rpos, rvel, 0.35)
        ev[k][3].record(st)
    torch.cuda.synchronize()
    f.check_flags()
    ph_ms = np.array([[ev[k][i].elapsed_time(ev[k][i + 1]) for i in range(3)] for k in range(n_ph)])
    ph_avg = ph_ms.mean(0)
    ph_counters = f.stats()
    # ---- e2e through the public API with host buffers (pinned H2D in, D2H pos/vel out)
    rpos_h = rpos.cpu().pin_memory()
    rvel_h = rvel.cpu().pin_memory()
    out_pos = torch.empty(f.pos_t.shape, dtype=torch.float64).pin_memory()
    out_vel = torch.empty(f.vel_t.shape, dtype=torch.float64).pin_memory()
    e2e_steps = min(args.steps, args.e2e_steps)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        rp = rpos_h.to(dev, non_blocking=True)
        rv = rvel_h.to(dev, non_blocking=True)
        resample_mix(k)
        f.step(rp, rv, 0.35, check=False)
        out_pos.copy_(f.pos_t, non_blocking=True)
        out_vel.copy_(f.vel_t, non_blocking=True)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    h2d = rpos_h.numel() * 8 * 2
    d2h = out_pos.numel() * 8 * 2

    # ---- multi-tick run (CrowdField.run, cw_crowd_run): the same ticks without a
    # per-tick barrier across envs, bit-identical to synchronous steps (tests/test_gpu_run.py).
    # Cannot host cfg5's per-step re-sampling (a host-driven scene swap between ticks).
    run = None
    if not args.no_run:
        f.run(2, rpos, rvel, 0.35)          # first-call attributes / scratch
        torch.cuda.synchronize()
        c0 = f.stats()
        flush.fill_(-1.0)                   # L2 flushed once; the grids read (>600 MB) exceed L2
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        run_resampled = 0
        with Clocks(dev.index) as rclk:
            r0.record(st)
            if CFG["resample"] > 0:
                # cfg5 driver: the same Bernoulli re-sampling schedule, run as
                # barrier-free segments between batched re-samples (envcore.run_with_resampling)
                from paper_2505_00690_b200.envcore import run_with_resampling
                run_resampled = run_with_resampling(sampler, f, env_seeds, counts, masks[:args.steps],
                                                    args.steps, rpos, rvel, 0.35)
            else:
                f.run(args.steps, rpos, rvel, 0.35)
            r1.record(st)
            torch.cuda.synchronize()
        run_ms = r0.elapsed_time(r1)
        rounds = int(_lib.lib().cw_crowd_run_rounds())
        launches = rounds + 3   # rounds + init + search server + finish
        if CFG["resample"] > 0:
            rs_ = f.last_run_stats
            # per window: init, server, finish + its rounds; per batched re-sample: the
            # sampling pipeline (~16 kernels incl. route anchors) + the respawn copies
            rounds = rs_["rounds"]
            launches = rs_["rounds"] + 3 * rs_["windows"] + 16 * rs_["sample_calls"]
        c1 = f.stats()
        # run-mode end to end: per call pinned H2D robot inputs, run(chunk), D2H pos/vel
        # (no re-sampling in this part: the timed run above carries the cfg5 driver)
        chunk = max(1, min(args.run_chunk, e2e_steps))
        n_chunks = max(1, e2e_steps // chunk)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n_chunks):
            rp = rpos_h.to(dev, non_blocking=True)
            rv = rvel_h.to(dev, non_blocking=True)
            f.run(chunk, rp, rv, 0.35, check=False)
            out_pos.copy_(f.pos_t, non_blocking=True)
            out_vel.copy_(f.vel_t, non_blocking=True)
        torch.cuda.synchronize()
        run_e2e_s = time.perf_counter() - t0
        f.check_flags()
        run = {"ms": run_ms, "rounds": rounds, "launches": launches, "clocks": rclk.summary(),
               "expansions": c1["astar_expansions"] - c0["astar_expansions"],
               "scanned": c1["path_points_scanned"] - c0["path_points_scanned"],
               "e2e_s": run_e2e_s, "e2e_ticks": n_chunks * chunk, "chunk": chunk, "resampled": run_resampled}

    # ---- full env step (crowd tick with the robot lane + robot step + reward + 128-ray
    # observations), the path the reference's perf harness times (harness.py:87-124)
    sb = measure_step_batch(b, f, dev, st, flush, min(args.steps, 200)) if not args.no_step_batch else None

    # ---- max over ranks; per-env stats all_gather (the one collective)
    stats = torch.stack([f.last_gap_t, b.obj_n.double(), b.walk_n.double(),
                         f.active_t.sum(1).double()], 1)
    tmax = torch.tensor([t_ms, sample_ms, e2e_s, run["ms"] if run else 0.0, run["e2e_s"] if run else 0.0],
                        dtype=torch.float64, device=dev)
    csum = shard.state_checksum(f.pos_t, f.vel_t, f.goal_t, f.last_gap_t)   # per env, exact
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        stats = shard.gather_env_stats(stats)
        csum = shard.gather_env_stats(csum[:, None])[:, 0]
    t_ms, sample_ms, e2e_s, run_ms_max, run_e2e_max = [float(x) for x in tmax.cpu()]
    if rank == 0:
        steps = args.steps
        env_steps = E * world * steps
        value = env_steps / (t_ms / 1e3)
        scenes = E * world / (sample_ms / 1e3)
        # roofline.  Whole dynamics step, SURVEY §8d byte model: 74 B per active
        # agent-step + 8 B per guidance path point scanned + 20 B per env-step (robot).
        bytes_step = (74.0 * active + 20.0 * E) + 8.0 * counters["path_points_scanned"] / steps
        avg_ms = t_ms / steps
        achieved = bytes_step / (avg_ms / 1e3) / 1e9
        peak, src = peaks()
        # per kernel (dominant one reported as `roofline`): k_guide = the §8d guidance
        # share (pos/goal/waypoint 40 B per agent + 8 B per path point); k_astar = 80 B
        # per expansion (8 neighbour g + passable, popped g); k_orca = the rest of §8d.
        exp_step = ph_counters["astar_expansions"] / n_ph
        scan_step = ph_counters["path_points_scanned"] / n_ph
        kb = {"k_guide": 40.0 * active + 8.0 * scan_step,
              "k_astar": 80.0 * exp_step,
              "k_orca": 34.0 * active + 20.0 * E}
        names = ["k_guide", "k_astar", "k_orca"]
        dom = names[int(np.argmax(ph_avg))]
        dom_ms = float(ph_avg[names.index(dom)])
        dom_ach = kb[dom] / (dom_ms / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "env-steps/s",
            "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "ms_per_step": round(avg_ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded procedural scenes)",
            "config": {"workload": f"{args.config}: {E} envs/GPU, {nx}x{nx} grid ({CFG['res']} m), "
                                   f"{CFG['objects']} objects, {CFG['peds']} pedestrians/env, {CFG['task']}, "
                                   f"neighbor_distance {CFG['nd']} m, dynamics step (+ scene sampling)"
                                   + (f", Bernoulli({CFG['resample']}) re-sampling inside each step"
                                      if CFG["resample"] else ""),
                       "envs_per_gpu": E, "grid": [nx, nx], "objects": CFG["objects"], "peds": CFG["peds"],
                       "resampled_envs": resampled,
                       "parallelism": f"env-shard x{world}", "l2": "flushed (256 MB write) between timed steps",
                       "robot": "static per env at a seeded walkable cell, zero velocity"},
            "scenes_per_sec": round(scenes, 1), "sample_ms_per_batch": round(sample_ms, 3),
            "sample_includes": "zones, WFC terrain, placement, raster + heightfield, nearest-obstacle map, "
                               "walk list, reach labels, A* move table, pedestrian spawn, route anchors",
            "resample_ms_per_step": round(resample_ms, 3),
            "agent_steps_per_sec": round(value * CFG["peds"], 1),
            "e2e": {"value": round(E * world * e2e_steps / e2e_s, 1), "unit": "env-steps/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "steps": e2e_steps},
            "roofline": {"bound": "hbm", "achieved": round(dom_ach, 3), "peak": peak, "unit": "GB/s",
                         "frac": round(dom_ach / peak, 7),
                         "traffic": args.traffic if args.traffic is not None else traffic_of(dom),
                         "traffic_source": "ncu --set full, profiles/r1_traffic.json (cfg2 tick 21)",
                         "kernel": dom, "peak_source": src, "bytes_per_launch": round(kb[dom], 1),
                         "avg_launch_ms": round(dom_ms, 4),
                         "note": "latency-bound serial search; measured per kernel in the synchronous tick "
                                 "(events around each launch); the multi-tick run overlaps the same device "
                                 "bodies, see roofline_step and profiles/r1_run_trace_cfg2.txt"},
            "roofline_step": {"bound": "hbm", "achieved": round(achieved, 3), "peak": peak, "unit": "GB/s",
                              "frac": round(achieved / peak, 7), "bytes_per_step": round(bytes_step, 1),
                              "model": "SURVEY 8d: 74 B/agent-step + 8 B/path point + 20 B/env-step"},
            "step_batch": sb,
            "kernels_ms": {n: round(float(v), 4) for n, v in zip(names, ph_avg)},
            "kernels_share": {n: round(float(v / ph_avg.sum()), 4) for n, v in zip(names, ph_avg)},
            "gpu_launches": 4 * steps,   # k_guide, k_astar, k_orca (two passes) per tick
            "clocks": clk.summary(),
            "counters": counters,
            "stats": {"min_gap": float(torch.nan_to_num(stats[:, 0], posinf=1e9).min()),
                      "mean_objects": float(stats[:, 1].mean()), "envs": int(stats.shape[0]),
                      # checksum of the per-env state checksums (pos, vel, goal, last gap after
                      # the whole bench) over all envs, and over the first E global envs --
                      # the latter is the same for every N (weak scaling, env-sharded)
                      "state_checksum": hex(shard.checksum_of(csum)),
                      "state_checksum_first_envs": hex(shard.checksum_of(csum[:E]))},
        }
        if run is not None and env_steps / (run_ms_max / 1e3) < line["value"]:
            run["slower"] = True   # e.g. cfg4: the synchronous tick stays the headline
            line["run"] = {"value": round(env_steps / (run_ms_max / 1e3), 1), "rounds": run["rounds"],
                           "what": "cw_crowd_run measured, slower than the synchronous tick here"}
            line["mode"] = "tick_sync"
            run = None
        if run is not None:
            # headline = the multi-tick run; the synchronous tick stays beside it
            line["mode"] = "run"
            line["tick_sync"] = {"value": line["value"], "ms_per_step": line["ms_per_step"],
                                 "e2e": line["e2e"], "l2": line["config"]["l2"], "clocks": line["clocks"],
                                 "gpu_launches": line["gpu_launches"],
                                 "what": "one CrowdField.step per tick (all envs, barrier per tick)"}
            run_val = env_steps / (run_ms_max / 1e3)
            run_avg = run_ms_max / steps
            bytes_run = (74.0 * active + 20.0 * E) + 8.0 * run["scanned"] / steps
            ach_run = bytes_run / (run_avg / 1e3) / 1e9
            line["value"] = round(run_val, 1)
            line["ms_per_step"] = round(run_avg, 4)
            line["agent_steps_per_sec"] = round(run_val * CFG["peds"], 1)
            line["config"]["workload"] += "; K ticks per CrowdField.run call (no per-tick barrier across envs)"
            line["config"]["l2"] = ("flushed (256 MB write) before the run; the per-env grids the step reads "
                                    "(labels, nearest, reach, moves: >600 MB) exceed the 126 MB L2")
            line["clocks"] = run["clocks"]
            line["gpu_launches"] = run["launches"]
            if not CFG["resample"]:   # cfg5 keeps the per-tick e2e (it carries the re-sampling)
                line["e2e"] = {"value": round(E * world * run["e2e_ticks"] / run_e2e_max, 1),
                               "unit": "env-steps/s",
                               "h2d_bytes_per_step": int(h2d / run["chunk"]),
                               "d2h_bytes_per_step": int(d2h / run["chunk"]), "steps": run["e2e_ticks"],
                               "what": f"CrowdField.run({run['chunk']}) with pinned host robot inputs copied in "
                                       f"and pos/vel copied out per call"}
            line["roofline_step"] = {"bound": "hbm", "achieved": round(ach_run, 3), "peak": peak,
                                     "unit": "GB/s", "frac": round(ach_run / peak, 7),
                                     "bytes_per_step": round(bytes_run, 1),
                                     "model": "SURVEY 8d: 74 B/agent-step + 8 B/path point + 20 B/env-step"}
            line["run"] = {"rounds": run["rounds"], "astar_expansions": run["expansions"],
                           "resampled_envs": run["resampled"],
                           "what": "cw_crowd_run: persistent A* server + ready-env ring + round kernels"
                                   + ("; cfg5 re-sampling: barrier-free 5-tick windows (cw_crowd_run_window) "
                                      "between batched re-samples of the envs that reached their re-sample tick"
                                      if CFG["resample"] else "")}
            if CFG["resample"]:
                line["config"]["resampled_envs"] = run["resampled"]
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline_sample(b, f, run_seeds)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def measure_step_batch(b, f, dev, st, flush, steps):
    """BatchedEnv.step_batch_device semantics on the bench batch: crowd tick with the
    robot lane (env_mask = live), then cw_robot_step (integrate, gating, contact,
    reward, observations); random actions resident on the device; L2 flushed."""
    import torch
    from paper_2505_00690_b200.robot import RobotBatch
    E = b.E
    rb = RobotBatch(b.labels, b.elev, float(b.params.res), "quadruped", horizon=10 ** 9)
    g = torch.Generator(device="cpu").manual_seed(7)
    wn = b.walk_n.long()
    pick = (torch.rand((E, 2), generator=g).to(dev) * wn[:, None].double()).long()
    cells = b.walk.gather(1, pick)
    nx = b.labels.shape[2]
    res = float(b.params.res)
    xy = lambda c: (((c % nx).double() + 0.5) * res, ((c // nx).double() + 0.5) * res)
    sx, sy = xy(cells[:, 0])
    gx, gy = xy(cells[:, 1])
    rb.set_state(sx, sy, torch.atan2(gy - sy, gx - sx), torch.stack([gx, gy], 1))
    acts = torch.rand((steps + 5, E, 2), generator=g).to(dev) * 2.0 - 1.0

    def tick(k):
        rp = torch.stack([rb.x, rb.y], -1)
        rv = torch.stack([rb.vx, rb.vy], -1)
        f.step(rp, rv, rb.model.body_radius, env_mask=rb.live().to(torch.uint8), check=False)
        rb.step(acts[k], (f.pos_t, f.radius_t, f.active_t))

    for k in range(5):
        tick(k)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for k in range(steps):
        flush.fill_(float(k))
        ev[k][0].record(st)
        tick(5 + k)
        ev[k][1].record(st)
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(c) for a, c in ev]))
    return {"value": round(E / (ms / 1e3), 1), "unit": "env-steps/s", "ms_per_step": round(ms, 4),
            "steps": steps, "robot": "quadruped",
            "what": "BatchedEnv.step_batch semantics: crowd tick with robot lane + robot step + reward + "
                    "128-ray depth fan + 16x10 height patch, device-resident actions, L2 flushed"}


def cpu_baseline_sample(b, f, run_seeds, n_env=12, warm=2, steps=40):
    """Oracle port (the reference's algorithm in numpy), 1 core, bounded sample:
    ``n_env`` envs of this config (GPU-sampled scenes, bit-identical to the
    oracle's), ``warm`` untimed ticks from spawn (every agent plans at tick 0),
    then ``steps`` timed ticks -- about 10-20 s of CPU work at cfg2."""
    from oracle import crowd as C
    grids = [(b.labels[i].cpu().numpy(), CFG["res"]) for i in range(n_env)]
    agents = []
    for i in range(n_env):
        k = b.sp_kind[i].cpu().numpy()
        agents.append(dict(pos=b.sp_pos[i].cpu().numpy(), goal=b.sp_goal[i].cpu().numpy(),
                           radius=np.array([C.RADIUS[x] for x in k]), pref=b.sp_pref[i].cpu().numpy(),
                           max_speed=np.array([C.MAX_SPEED[x] for x in k]), kind=k))
    ref = C.CrowdFieldOracle(grids, C.Config(neighbor_distance=CFG["nd"]), [int(s) for s in run_seeds[:n_env]])
    ref.set_agents(agents)
    for _ in range(warm):
        ref.step()
    t0 = time.perf_counter()
    for _ in range(steps):
        ref.step()
    dt = time.perf_counter() - t0
    return {"value": round(n_env * steps / dt, 3), "unit": "env-steps/s", "cores": 1,
            "kind": "port", "seconds": round(dt, 2),
            "sample": f"{n_env} envs of this config, {warm} untimed + {steps} timed crowd ticks from spawn, "
                      f"oracle port (numpy restatement of the reference), 1 thread"}


# ============================================================================ reference arm
def _ref_worker(args):
    """One process: generate its env with the oracle, then time `steps` ticks."""
    env_id, steps, warm, cfg = args
    from oracle import crowd as C
    from oracle import scene as S
    from oracle.rng import child_seed
    import json as _json
    cat = S.load_catalog_tuples(_json.load(open(os.path.join(ROOT, "paper_2505_00690_b200", "data", "catalog.json"))))
    from oracle import routes as R
    s = child_seed(0, "env", env_id)
    spec = make_spec(cfg)
    # one env sample as BatchedEnv builds it: generate_scene (incl. raster and the
    # route anchors, scene.py:38-90), crowd spawn (step.py:37) and _prepare_env
    # (nearest-obstacle BFS, field.py:60-67)
    ts = time.perf_counter()
    sc = S.generate_scene(dict(seed=s, extent=spec.extent_m, res=cfg["res"], task=cfg["task"], split="Train",
                               density=spec.object_density, mix=MIX), cat)
    R.sample_route_anchors(sc["labels"], cfg["res"], s, spec.extent_m, cfg["task"])
    sp = C.spawn_agents(sc["labels"], cfg["res"], cfg["peds"], child_seed(s, "crowd", 0))
    f = C.CrowdFieldOracle([(sc["labels"], cfg["res"])], C.Config(neighbor_distance=cfg["nd"]),
                           [child_seed(s, "crowd-run")])
    t_scene = time.perf_counter() - ts
    f.set_agents([sp])
    for _ in range(warm):
        f.step()
    t = []
    for _ in range(steps):
        t0 = time.perf_counter()
        f.step()
        t.append(time.perf_counter() - t0)
    return t, t_scene


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    # bounded: one env per core, at most a few minutes for the whole --steps/--warmup run
    steps = max(1, min(args.steps, 60))
    warm = max(0, min(args.warmup, 5))
    with mp.get_context("spawn").Pool(cores) as pool:
        t0 = time.perf_counter()
        res = pool.map(_ref_worker, [(i, steps, warm, dict(CFG)) for i in range(cores)])
        wall = time.perf_counter() - t0
    times = [r[0] for r in res]
    t_scene = max(r[1] for r in res)                 # all cores sample one scene each, in parallel
    per_step = np.max(np.array(times), axis=0)       # all cores step in parallel
    total = float(per_step.sum())
    value = cores * steps / total
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "env-steps/s",
            "n_gpus": world, "steps": steps, "warmup": warm,
            "ms_per_step": round(1e3 * total / steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded procedural scenes)",
            "config": {"workload": f"{args.config} shape: {CFG['extent']} m at {CFG['res']} m, "
                                   f"{CFG['objects']} objects, {CFG['peds']} peds/env; sample of one env per host core",
                       "envs": cores, "parallelism": f"{cores} processes"},
            "cpu_baseline": {"value": round(value, 3), "unit": "env-steps/s", "cores": cores,
                             "kind": "port",
                             "sample": f"{cores} {args.config} envs (one per core) x {steps} crowd ticks; "
                                       f"oracle port of the reference algorithm; wall {wall:.1f}s incl. scene gen"},
            "e2e": {"value": round(value, 3), "unit": "env-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "scenes_per_sec": round(cores / t_scene, 4),
            "sample_includes": "generate_scene (zones, WFC terrain, placement, raster + heightfield), route "
                               "anchors, crowd spawn, nearest-obstacle map; one scene per core"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--envs", type=int, default=None)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--threads", type=int, default=128)
    ap.add_argument("--sample-warmup", type=int, default=1)
    ap.add_argument("--sample-reps", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-step-batch", action="store_true")
    ap.add_argument("--no-run", action="store_true",
                    help="headline from synchronous ticks only (skip the CrowdField.run measurement)")
    ap.add_argument("--run-chunk", type=int, default=25,
                    help="ticks per CrowdField.run call in the run-mode e2e measurement")
    ap.add_argument("--phase-steps", type=int, default=100)
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch of the dominant kernel from an ncu --set full capture")
    args = ap.parse_args()
    CFG.clear()
    CFG.update(CONFIGS[args.config])
    if args.envs is None:
        args.envs = CFG["envs"]
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

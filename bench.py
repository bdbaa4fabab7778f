"""Benchmark: async scene sampling + crowd dynamics step on B200 (BASELINE.json configs[1]).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfgX]

Workload (cfg2, the default): E=1024 envs per GPU, 32 m x 32 m at 0.125 m (256x256
grid), 64 objects, 32 pedestrians per env, NavDynamic, terrain mix 0.25 each, dt 0.05,
seeds child_seed(0, "env", global_env_id).  A "step" is one crowd tick of every env
of the rank.  ``value`` = K consecutive ticks through ``CrowdField.run`` (no per-tick
barrier across envs, bit-identical to K ``CrowdField.step`` calls); ``e2e`` = the
reference's per-tick API, one ``CrowdField.step`` per tick with the robot inputs
copied in from pinned host memory and pos/vel read back to the host every tick.
Scenes/s is the whole ``cw_sample_scenes`` pipeline over the same E envs.

``--gpus N`` (N > 1) without torchrun re-launches itself under
``torch.distributed.run`` with N ranks; each rank owns E envs (weak scaling, no
data-path collective; one all_gather of per-env stats at the end).

``--impl reference`` times the reference's CPU implementation of the same path on
the host cores: the unmodified reference (``baseline/_ref``) when installed, else the
oracle port; one env per process, the same tick window (W untimed + K timed ticks
from spawn) and the same static robot as our arm.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
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
ROBOT_SEED = 1234     # static robot: torch.Generator(cpu).manual_seed(ROBOT_SEED + rank)
REF_BUDGET_S = 150.0  # CPU arms: stop timing ticks after this long per process (bounded sample)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_of(config, kernel):
    """dram read+write bytes per launch of `kernel` from this config's committed
    ncu --set full capture (profiles/r2_traffic_<config>.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", f"r2_traffic_{config}.json")) as fh:
            d = json.load(fh)
        k = d["kernels"][kernel]
        return float(k["dram_read_bytes"] + k["dram_write_bytes"]), d.get("source", "")
    except Exception:
        return None, None


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def host_cores():
    try:
        import psutil
        phys = psutil.cpu_count(logical=False)
    except Exception:
        phys = None
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = os.cpu_count() or 1
    return usable, phys


class Clocks:
    """NVML clocks + throttle reasons sampled every 2 ms on a thread (B200_PROFILING
    clocks line).  ``summary(t0, t1)`` reports the samples inside the timed window
    widened to at least ``min_span`` seconds around it (the GPU is busy with the
    bench's other passes on both sides)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, gpu):
        self.rows = []
        self.stop = threading.Event()
        self.err = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            # NVML enumerates all GPUs; CUDA_VISIBLE_DEVICES may remap
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[gpu]) if vis and vis.split(",")[gpu].strip().isdigit() else gpu
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception as exc:   # no NVML
            self.nv = None
            self.err = str(exc)[:80]
        self.th = threading.Thread(target=self._loop, daemon=True)

    def _loop(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                self.rows.append((time.perf_counter(), float(sm), int(rs), int(util)))
            except Exception as exc:
                self.err = str(exc)[:80]
            time.sleep(0.002)

    def start(self):
        if self.nv is not None:
            self.th.start()
        return self

    def close(self):
        self.stop.set()
        if self.th.is_alive():
            self.th.join()

    def summary(self, t0, t1, min_span=1.0):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        pad = max(0.0, (min_span - (t1 - t0)) / 2)
        rows = [r for r in self.rows if t0 - pad <= r[0] <= t1 + pad]
        inside = sum(1 for r in rows if t0 <= r[0] <= t1)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_sm, "reasons": [], "samples": 0}
        reasons = sorted({n for r in rows for n, b in self.REASONS.items() if r[2] & b})
        return {"sm_mhz": float(np.median([r[1] for r in rows])), "sm_max_mhz": self.max_sm,
                "reasons": reasons, "samples": len(rows), "samples_in_timed_region": inside,
                "window_s": round(max(t1 - t0, min_span), 3), "source": "NVML, 2 ms sampling",
                "gpu_util_median": float(np.median([r[3] for r in rows]))}


def make_spec(cfg=None):
    from paper_2505_00690_b200.urbangen import SceneSpec, TaskKind
    cfg = cfg or CFG
    return SceneSpec(seed=0, extent_m=(cfg["extent"], cfg["extent"]), task_kind=TaskKind(cfg["task"]),
                     object_density=density(cfg), pedestrian_count=cfg["peds"],
                     terrain_mix=MIX, grid_resolution_m=cfg["res"])


def density(cfg):
    n = int(np.ceil(cfg["extent"] / cfg["res"]))
    base = int(np.floor(4.0 * (n * n * cfg["res"] * cfg["res"]) / 100.0 + 0.5))  # 41 at 32 m
    return cfg["objects"] / base if cfg["objects"] else 0.0


def robot_picks(E, rank):
    """The static robot's walk-list index fraction per env (shared by both arms)."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(ROBOT_SEED + rank)
    return torch.rand(E, generator=g).double()


# ============================================================================ ours
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2505_00690_b200 import _lib
    from paper_2505_00690_b200.crowd import CrowdConfig, CrowdField
    from paper_2505_00690_b200.rng import child_seeds_device
    from paper_2505_00690_b200.urbangen import SceneSampler

    rank, world, local = dist_env()
    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", local % max(ndev, 1))
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group(args.backend)
    _lib.build()
    from paper_2505_00690_b200 import shard
    clk = Clocks(dev.index).start()
    E = args.envs
    spec = make_spec()
    nx = int(np.ceil(CFG["extent"] / CFG["res"]))
    N = nx * nx
    zero = torch.zeros(E, dtype=torch.int64, device=dev)
    gids = torch.from_numpy(shard.env_ids(rank, world, E)).to(dev)   # rank owns [r*E, (r+1)*E)
    env_seeds = child_seeds_device(zero, "env", gids)
    crowd_seeds = child_seeds_device(env_seeds, "crowd", 0)
    run_seeds = child_seeds_device(env_seeds, "crowd-run").cpu().numpy().view(np.uint64)
    sampler = SceneSampler(spec, E, device=dev)
    st = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)

    # ---- scene sampling throughput (whole pipeline, E envs per launch sequence)
    for _ in range(max(1, args.sample_warmup)):
        sampler.sample(env_seeds, crowd_seeds, check=False)
    torch.cuda.synchronize()
    sampler.batch.check_status()
    s0, s1 = ev(), ev()
    reps = args.sample_reps
    s0.record(st)
    for _ in range(reps):
        sampler.sample(env_seeds, crowd_seeds, check=False)
    s1.record(st)
    torch.cuda.synchronize()
    sample_ms = s0.elapsed_time(s1) / reps
    b = sampler.batch
    b.check_status()
    walk_total = float(b.walk_n.double().sum())

    # ---- crowd
    f = CrowdField(b, CrowdConfig(neighbor_distance=CFG["nd"]), [int(s) for s in run_seeds], device=dev,
                   threads=args.threads)
    f.set_from_spawn(b)
    f.prepare_step()
    # robot: static at a seeded walkable cell per env, zero velocity (same in --impl reference)
    pick = (robot_picks(E, rank).to(dev) * b.walk_n.double()).long()
    cell = b.walk.gather(1, pick[:, None])[:, 0].long()
    rpos = torch.stack([((cell % nx).double() + 0.5) * CFG["res"],
                        ((cell // nx).double() + 0.5) * CFG["res"]], dim=1).contiguous()
    rvel = torch.zeros_like(rpos)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MB > L2
    active = int(f.active_t.sum().item())
    resampled = 0
    counts = torch.zeros(E, dtype=torch.int64, device=dev)
    masks = []
    if CFG["resample"] > 0:
        # cfg5 driver: env i re-sampled at step t iff
        # make_rng(0, "resample-mix", t).random(E) < p, via BatchedEnv.reset semantics
        from paper_2505_00690_b200.rng import child_seed as _cs
        T_all = args.warmup + args.steps
        masks = [np.flatnonzero(np.random.Generator(np.random.PCG64(_cs(0, "resample-mix", k)))
                                .random(E * world)[rank * E:(rank + 1) * E] < CFG["resample"])
                 for k in range(T_all)]

    standby = None   # per-tick loops: asynchronous scene sampling (envcore.SceneStandby)

    def resample_mix(k):
        nonlocal resampled
        if CFG["resample"] > 0 and masks[k].size:
            sl = torch.from_numpy(masks[k]).to(dev)
            counts[sl] += 1
            if standby is not None:   # the rows' next scenes (and first replans) sampled ahead
                standby.take(masks[k])   # + set_from_spawn
            else:
                env_k = env_seeds[sl]
                new_scene = child_seeds_device(env_k, "resample", counts[sl])
                sampler.sample(new_scene, child_seeds_device(env_k, "crowd", counts[sl]), slots=sl, check=False)
                f.set_from_spawn(b, rows=sl)
            resampled += int(masks[k].size)

    # ---- value: ticks W .. W+K from spawn through CrowdField.run (the same ticks,
    # no per-tick barrier across envs; bit-identical to K synchronous steps)
    for k in range(args.warmup):
        resample_mix(k)
        if k >= args.warmup - 2 and args.mode == "run" and not CFG["resample"]:
            f.run(1, rpos, rvel, 0.35, check=False)   # first-call setup of the run path, untimed
        else:
            f.step(rpos, rvel, 0.35, check=False)
    torch.cuda.synchronize()
    f.check_flags()
    f.counters_t.zero_()
    flush.fill_(-1.0)                   # L2 flushed once; the grids read (>600 MB) exceed L2
    r0, r1 = ev(), ev()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    run_resampled = 0
    prof_range = bool(os.environ.get("CW_PROFILE_RANGE"))   # ncu --replay-mode app-range window
    if prof_range:
        torch.cuda.profiler.start()
    t_run0 = time.perf_counter()
    r0.record(st)
    if CFG["resample"] > 0:
        # cfg5 driver: the same Bernoulli re-sampling schedule, run as barrier-free
        # segments between batched re-samples (envcore.run_with_resampling)
        from paper_2505_00690_b200.envcore import run_with_resampling
        run_resampled = run_with_resampling(sampler, f, env_seeds, counts, masks[args.warmup:], args.steps,
                                            rpos, rvel, 0.35)
    elif args.mode == "run":
        f.run(args.steps, rpos, rvel, 0.35)
    else:
        for k in range(args.steps):
            f.step(rpos, rvel, 0.35, check=False)
    r1.record(st)
    torch.cuda.synchronize()
    t_run1 = time.perf_counter()
    if prof_range:
        torch.cuda.profiler.stop()
    f.check_flags()
    run_ms = r0.elapsed_time(r1)
    c_run = f.stats()
    if CFG["resample"] > 0:
        rs_ = f.last_run_stats
        # per window: init, server, finish + its rounds; per batched re-sample: the
        # sampling pipeline (~17 kernels incl. route anchors) + the respawn copies
        launches = rs_["rounds"] + rs_["servers"] + 2 * rs_["windows"] + 17 * rs_["sample_calls"]
        rounds = rs_["rounds"]
    elif args.mode == "run":
        rounds = int(_lib.lib().cw_crowd_run_rounds())
        launches = rounds + int(_lib.lib().cw_crowd_run_servers()) + 2   # rounds + servers + init + finish
    else:
        rounds = 0
        launches = 4 * args.steps
    csum_value = shard.state_checksum(f.pos_t, f.vel_t, f.goal_t, f.last_gap_t)   # per env, exact

    # the per-tick loops re-sample through the standby pool: each reset installs a scene
    # sampled ahead (same seeds) and starts sampling the row's next one beside the ticks;
    # the pool's initial fill (every row's next scene) is setup, outside the timed regions
    if CFG["resample"] > 0 and not args.no_standby:
        from paper_2505_00690_b200.envcore import SceneStandby
        standby = SceneStandby(sampler, env_seeds, counts, field=f)
        torch.cuda.synchronize()

    # ---- synchronous tick (CrowdField.step, barrier per tick), L2 flushed between ticks
    n_sync = min(args.steps, args.sync_steps)
    starts = [ev() for _ in range(n_sync)]
    ends = [ev() for _ in range(n_sync)]
    f.counters_t.zero_()
    torch.cuda.synchronize()
    t_sync0 = time.perf_counter()
    for k in range(n_sync):
        flush.fill_(float(k))          # untimed
        starts[k].record(st)
        if masks:
            resample_mix((args.warmup + k) % len(masks))   # cfg5: the re-sampling is part of the step
        f.step(rpos, rvel, 0.35, check=False)
        ends[k].record(st)
    torch.cuda.synchronize()
    t_sync1 = time.perf_counter()
    f.check_flags()
    sync_ms = float(np.mean([s.elapsed_time(e) for s, e in zip(starts, ends)]))
    c_sync = f.stats()

    # ---- per-kernel pass (same stream, events between the three launches)
    n_ph = min(args.steps, args.phase_steps)
    pev = [[ev() for _ in range(4)] for _ in range(n_ph)]
    f.counters_t.zero_()
    torch.cuda.synchronize()
    for k in range(n_ph):
        flush.fill_(float(k))
        pev[k][0].record(st)
        f.step_phase(1, rpos, rvel, 0.35)
        pev[k][1].record(st)
        f.step_phase(2, rpos, rvel, 0.35)
        pev[k][2].record(st)
        f.step_phase(4, rpos, rvel, 0.35)
        pev[k][3].record(st)
    torch.cuda.synchronize()
    f.check_flags()
    ph_ms = np.array([[pev[k][i].elapsed_time(pev[k][i + 1]) for i in range(3)] for k in range(n_ph)])
    ph_avg = ph_ms.mean(0)
    ph_counters = f.stats()

    # ---- e2e through the reference's per-tick API (CrowdField.step): every tick the
    # robot inputs come from pinned host memory and pos/vel are read back to the host
    # (stream synchronised before the next tick, as a closed-loop caller does)
    rpos_h = rpos.cpu().pin_memory()
    rvel_h = rvel.cpu().pin_memory()
    out_pos = torch.empty(f.pos_t.shape, dtype=torch.float64).pin_memory()
    out_vel = torch.empty(f.vel_t.shape, dtype=torch.float64).pin_memory()
    e2e_steps = min(args.steps, args.e2e_steps)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        rp = rpos_h.to(dev, non_blocking=True)
        rv = rvel_h.to(dev, non_blocking=True)
        if masks:
            resample_mix((args.warmup + k) % len(masks))   # cfg5: the re-sampling is part of the step
        f.step(rp, rv, 0.35, check=False)
        out_pos.copy_(f.pos_t, non_blocking=True)
        out_vel.copy_(f.vel_t, non_blocking=True)
        st.synchronize()
    e2e_s = time.perf_counter() - t0
    h2d = rpos_h.numel() * 8 * 2
    d2h = out_pos.numel() * 8 * 2

    # ---- e2e of the multi-tick API: CrowdField.run(chunk) calls, inputs in / pos, vel out per call
    run_e2e = None
    if not CFG["resample"] and args.mode == "run":
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
            st.synchronize()
        run_e2e = (time.perf_counter() - t0, n_chunks * chunk, chunk)
        f.check_flags()

    # ---- full env step (crowd tick with the robot lane + robot step + reward + 128-ray
    # observations), the path the reference's perf harness times (harness.py:87-124)
    sb = measure_step_batch(b, f, dev, st, flush, min(args.steps, 200)) if not args.no_step_batch else None
    clk.close()

    # ---- max over ranks; per-env stats all_gather (the one collective)
    stats = torch.stack([f.last_gap_t, b.obj_n.double(), b.walk_n.double(),
                         f.active_t.sum(1).double()], 1)
    tmax = torch.tensor([run_ms, sample_ms, e2e_s, sync_ms, run_e2e[0] if run_e2e else 0.0],
                        dtype=torch.float64, device=dev)
    comm_ok = True
    if world > 1:
        tmax = shard.max_tensor_over_ranks(tmax)
        stats = shard.gather_env_stats(stats)
        csum_value = shard.gather_env_stats(csum_value[:, None])[:, 0]
        comm_ok = int(stats.shape[0]) == E * world
    run_ms, sample_ms, e2e_s, sync_ms, run_e2e_s = [float(x) for x in tmax.cpu()]
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    steps = args.steps
    env_steps = E * world * steps
    value = env_steps / (run_ms / 1e3)
    avg_ms = run_ms / steps
    scenes = E * world / (sample_ms / 1e3)
    peak, peak_src = peaks()
    # roofline, dominant kernel of the synchronous tick.  Algorithmic bytes per launch, with
    # the state in float64 (the dtype the path computes in; SURVEY 8d sized it for fp32):
    #   k_guide = 57 B/agent (active 1, goal 16, pos 16, path head + count 8 in; waypoint
    #             16 out) + 4 B per path point read (int32 cell) + 1 B per line-of-sight
    #             label sample;
    #   k_astar = 80 B per expansion (popped g, 8 neighbour g + move byte);
    #   k_orca  = 126 B/agent (pos, vel, goal, waypoint 16 each, pref, radius, max_speed 8
    #             each, active 1 in; pos, vel 16 each out; nearest 4 + label 1 at the agent's
    #             cells) + 80 B/env (robot pos + vel 32, PCG64 stream 48).
    exp_step = ph_counters["astar_expansions"] / n_ph
    pts_step = ph_counters["path_points_read"] / n_ph
    los_step = ph_counters["los_samples_read"] / n_ph
    kb = {"k_guide": 57.0 * active + 4.0 * pts_step + 1.0 * los_step,
          "k_astar": 80.0 * exp_step,
          "k_orca": 126.0 * active + 80.0 * E}
    names = ["k_guide", "k_astar", "k_orca"]
    dom = names[int(np.argmax(ph_avg))]
    dom_ms = float(ph_avg[names.index(dom)])
    dom_ach = kb[dom] / (dom_ms / 1e3) / 1e9
    traffic, tsrc = traffic_of(args.config, dom)
    if args.traffic is not None:
        traffic, tsrc = args.traffic, "--traffic"
    # whole step (SURVEY 8d's fields at float64): per active agent-step read pos, vel, goal,
    # waypoint 16 each, pref, radius, max_speed 8 each, active 1, path head + count 8 (97 B),
    # write pos, vel, waypoint 16 each + path head + count 8 (56 B), grid lookups 5 B
    # -> 158 B; per env-step 80 B (robot, PCG64 stream); plus the guidance reads the device
    # makes (4 B per path point, 1 B per LOS sample; device counters)
    def step_bytes(c, n):
        return 158.0 * active + 80.0 * E + (4.0 * c["path_points_read"] + 1.0 * c["los_samples_read"]) / n
    bytes_run = step_bytes(c_run, steps)
    ach_run = bytes_run / (avg_ms / 1e3) / 1e9
    bytes_sync = step_bytes(c_sync, n_sync)
    # sampling: elev 4N + labels N + nearest 4N + walk list 4W + agents 40A per env
    bytes_sample = E * (9.0 * N + 40.0 * CFG["peds"]) + 4.0 * walk_total
    ach_sample = bytes_sample / (sample_ms / 1e3) / 1e9
    workload = (f"{args.config}: {E} envs/GPU, {nx}x{nx} grid ({CFG['res']} m), {CFG['objects']} objects, "
                f"{CFG['peds']} pedestrians/env, {CFG['task']}, neighbor_distance {CFG['nd']} m; "
                f"ticks {args.warmup}..{args.warmup + steps} from spawn"
                + (f"; Bernoulli({CFG['resample']}) re-sampling inside each step" if CFG["resample"] else ""))
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "env-steps/s",
        "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": round(avg_ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded procedural scenes)",
        "mode": args.mode if not CFG["resample"] else "run_windows",
        "config": {"workload": workload, "envs_per_gpu": E, "grid": [nx, nx], "objects": CFG["objects"],
                   "peds": CFG["peds"], "parallelism": f"env-shard x{world} ({args.backend})",
                   "l2": "flushed (256 MB write) before the timed run; the per-env grids it reads "
                         "(labels, nearest, reach, moves: >600 MB at cfg2) exceed the 126 MB L2",
                   "robot": "static per env at a seeded walkable cell, zero velocity",
                   "resampled_envs": run_resampled or resampled},
        "what": ("CrowdField.run(K): K ticks of every env without a per-tick barrier across envs "
                 "(persistent A* server + ready-env ring + round kernels), bit-identical to K "
                 "CrowdField.step calls" if args.mode == "run" else "K CrowdField.step calls"),
        "e2e": {"value": round(E * world * e2e_steps / e2e_s, 1), "unit": "env-steps/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
                "what": "the reference's per-tick API: CrowdField.step once per tick (cfg5: after the "
                        "tick's Bernoulli re-sampling); robot pos/vel copied in from pinned host memory "
                        "and crowd pos/vel read back to the host every tick (stream synchronised per tick)"},
        "tick_sync": {"value": round(E * world / (sync_ms / 1e3), 1), "ms_per_step": round(sync_ms, 4),
                      "steps": n_sync, "l2": "flushed (256 MB write) between timed ticks",
                      "clocks": clk.summary(t_sync0, t_sync1),
                      "what": "one CrowdField.step per tick (cfg5: after the tick's re-sampling), "
                              "device-resident inputs (events per tick)"},
        "scenes_per_sec": round(scenes, 1), "sample_ms_per_batch": round(sample_ms, 3),
        "sample_includes": "zones, WFC terrain, placement, raster + heightfield, nearest-obstacle map, "
                           "walk list, reach labels, A* move table, pedestrian spawn, route anchors",
        "agent_steps_per_sec": round(value * CFG["peds"], 1),
        "roofline": {"bound": "hbm", "achieved": round(dom_ach, 3), "peak": peak, "unit": "GB/s",
                     "frac": round(dom_ach / peak, 7), "traffic": traffic, "traffic_source": tsrc,
                     "kernel": dom, "peak_source": peak_src, "bytes_per_launch": round(kb[dom], 1),
                     "avg_launch_ms": round(dom_ms, 4),
                     "bytes_model": {"k_guide": "57 B/agent + 4 B/path point read + 1 B/LOS sample",
                                     "k_astar": "80 B/expansion", "k_orca": "126 B/agent + 80 B/env",
                                     "state": "float64"},
                     "note": "dominant kernel of the synchronous tick (events around each launch on the "
                             "launching stream); a latency-bound serial search"},
        "roofline_step": {"bound": "hbm", "achieved": round(ach_run, 3), "peak": peak, "unit": "GB/s",
                          "frac": round(ach_run / peak, 7), "bytes_per_step": round(bytes_run, 1),
                          "bytes_per_step_sync": round(bytes_sync, 1),
                          "model": "SURVEY 8d fields at float64: 158 B/agent-step + 80 B/env-step + the "
                                   "guidance reads made (4 B/path point, 1 B/LOS sample; device counters)"},
        "roofline_sampling": {"bound": "hbm", "achieved": round(ach_sample, 3), "peak": peak, "unit": "GB/s",
                              "frac": round(ach_sample / peak, 7), "bytes_per_batch": round(bytes_sample, 1),
                              "model": "SURVEY 8d: 9N + 4W + 40A bytes per env-sample (elev, labels, "
                                       "nearest, walk list, agents)"},
        "step_batch": sb,
        "kernels_ms": {n: round(float(v), 4) for n, v in zip(names, ph_avg)},
        "kernels_share": {n: round(float(v / ph_avg.sum()), 4) for n, v in zip(names, ph_avg)},
        "gpu_launches": int(launches),
        "run": {"rounds": rounds, "astar_expansions": c_run["astar_expansions"],
                "path_points_read": c_run["path_points_read"], "los_samples_read": c_run["los_samples_read"]},
        "clocks": clk.summary(t_run0, t_run1),
        "counters_sync": c_sync,
        "stats": {"min_gap": float(torch.nan_to_num(stats[:, 0], posinf=1e9).min()),
                  "mean_objects": float(stats[:, 1].mean()), "envs": int(stats.shape[0]),
                  "comm_nranks_ok": comm_ok,
                  # checksum of the per-env state checksums (pos, vel, goal, last gap right
                  # after the timed ticks) over all envs and over the first E global envs --
                  # the latter is the same for every N (weak scaling, env-sharded)
                  "state_checksum": hex(shard.checksum_of(csum_value)),
                  "state_checksum_first_envs": hex(shard.checksum_of(csum_value[:E]))},
    }
    if run_e2e is not None:
        line["e2e_run"] = {"value": round(E * world * run_e2e[1] / run_e2e_s, 1), "unit": "env-steps/s",
                           "h2d_bytes_per_step": int(h2d / run_e2e[2]), "d2h_bytes_per_step": int(d2h / run_e2e[2]),
                           "steps": run_e2e[1],
                           "what": f"CrowdField.run({run_e2e[2]}) calls, pinned host robot inputs in and "
                                   f"pos/vel out per call"}
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(args)
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


# ============================================================================ CPU arms
def _reference_available():
    return os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "citywalk"))


def _ref_worker(job):
    """One process, one env (global id ``env_id``): sample it as BatchedEnv does
    (generate_scene incl. raster and route anchors, spawn_agents, CrowdField prep),
    then W untimed + K timed crowd ticks with the bench's static robot."""
    env_id, steps, warm, cfg, use_ref, robot_u = job
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    if use_ref:
        sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
        from citywalk.crowd import CrowdConfig, CrowdField, spawn_agents
        from citywalk.rng import child_seed
        from citywalk.urbangen import SceneSpec, TaskKind, generate_scene, rasterize_occupancy
        s = child_seed(0, "env", env_id)
        ts = time.perf_counter()
        spec = SceneSpec(seed=s, extent_m=(cfg["extent"], cfg["extent"]), task_kind=TaskKind(cfg["task"]),
                         object_density=density(cfg), pedestrian_count=cfg["peds"], terrain_mix=MIX,
                         grid_resolution_m=cfg["res"])
        occ = rasterize_occupancy(generate_scene(spec))
        agents = spawn_agents(occ, cfg["peds"], child_seed(s, "crowd", 0))
        f = CrowdField([occ], CrowdConfig(neighbor_distance=cfg["nd"]), [child_seed(s, "crowd-run")])
        t_scene = time.perf_counter() - ts
        f.set_agents([agents])
        labels = occ.labels
    else:
        import json as _json
        from oracle import crowd as C
        from oracle import routes as R
        from oracle import scene as S
        from oracle.rng import child_seed
        cat = S.load_catalog_tuples(_json.load(open(os.path.join(ROOT, "paper_2505_00690_b200", "data",
                                                                 "catalog.json"))))
        s = child_seed(0, "env", env_id)
        ts = time.perf_counter()
        ext = (cfg["extent"], cfg["extent"])
        sc = S.generate_scene(dict(seed=s, extent=ext, res=cfg["res"], task=cfg["task"], split="Train",
                                   density=density(cfg), mix=MIX), cat)
        R.sample_route_anchors(sc["labels"], cfg["res"], s, ext, cfg["task"])
        sp = C.spawn_agents(sc["labels"], cfg["res"], cfg["peds"], child_seed(s, "crowd", 0))
        f = C.CrowdFieldOracle([(sc["labels"], cfg["res"])], C.Config(neighbor_distance=cfg["nd"]),
                               [child_seed(s, "crowd-run")])
        t_scene = time.perf_counter() - ts
        f.set_agents([sp])
        labels = sc["labels"]
    walk = np.flatnonzero(labels.reshape(-1) == 2)
    c = int(walk[int(robot_u * len(walk))])
    nx = labels.shape[1]
    rp = np.array([[(c % nx + 0.5) * cfg["res"], (c // nx + 0.5) * cfg["res"]]])
    rv = np.zeros((1, 2))
    t_start = time.perf_counter()
    for _ in range(warm):
        f.step(robot_pos=rp, robot_vel=rv, robot_radius=0.35)
    t = []
    for _ in range(steps):
        t0 = time.perf_counter()
        f.step(robot_pos=rp, robot_vel=rv, robot_radius=0.35)
        t.append(time.perf_counter() - t0)
        if t0 - t_start > REF_BUDGET_S:   # bounded sample (e.g. cfg4: seconds per tick)
            break
    return t, t_scene


def _cpu_pool(n_env, steps, warm, use_ref):
    import multiprocessing as mp
    u = robot_picks(max(n_env, 1), 0).numpy()
    jobs = [(i, steps, warm, dict(CFG), use_ref, float(u[i])) for i in range(n_env)]
    with mp.get_context("spawn").Pool(n_env) as pool:
        t0 = time.perf_counter()
        res = pool.map(_ref_worker, jobs)
        wall = time.perf_counter() - t0
    k = min(len(r[0]) for r in res)                   # ticks every process completed
    times = np.array([r[0][:k] for r in res])
    t_scene = max(r[1] for r in res)                 # all processes sample one scene each, in parallel
    total = float(np.max(times, axis=0).sum())       # all processes step in parallel
    return n_env * k / total, total, t_scene, wall, k


def cpu_baseline(args):
    """Bounded CPU sample beside our line: the reference (or the port) on all host
    cores, one env per process, W untimed + a few timed ticks of the bench window."""
    usable, phys = host_cores()
    use_ref = _reference_available()
    steps = max(1, min(args.steps, args.cpu_steps))
    warm = min(args.warmup, 60)
    v, total, t_scene, wall, steps = _cpu_pool(usable, steps, warm, use_ref)
    return {"value": round(v, 3), "unit": "env-steps/s", "cores": usable, "physical_cores": phys,
            "kind": "reference" if use_ref else "port", "seconds": round(total, 2),
            "scenes_per_sec": round(usable / t_scene, 4),
            "sample": f"{usable} {args.config} envs (one per process, global ids 0..{usable - 1}), {warm} untimed + "
                      f"{steps} timed crowd ticks from spawn with the bench's static robot; "
                      + ("unmodified reference (baseline/_ref)" if use_ref else "oracle port") +
                      f"; wall {wall:.1f}s incl. scene sampling"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    usable, phys = host_cores()
    use_ref = _reference_available()
    # the same tick window as our arm (W untimed + K timed from spawn), bounded so the
    # whole run stays within a few minutes
    warm = min(args.warmup, 100)
    steps = max(1, min(args.steps, args.ref_steps))
    v, total, t_scene, wall, steps = _cpu_pool(usable, steps, warm, use_ref)
    kind = "reference" if use_ref else "port"
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 3), "unit": "env-steps/s",
            "n_gpus": world, "steps": steps, "warmup": warm,
            "ms_per_step": round(1e3 * total / steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded procedural scenes)",
            "config": {"workload": f"{args.config} shape: {CFG['extent']} m at {CFG['res']} m, {CFG['objects']} "
                                   f"objects, {CFG['peds']} peds/env, neighbor_distance {CFG['nd']} m; one env per "
                                   f"host process (global ids 0..{usable - 1}); ticks {warm}..{warm + steps} "
                                   f"from spawn, static robot as in our arm",
                       "envs": usable, "parallelism": f"{usable} processes"},
            "cpu_baseline": {"value": round(v, 3), "unit": "env-steps/s", "cores": usable, "physical_cores": phys,
                             "kind": kind,
                             "sample": f"{usable} {args.config} envs x {steps} timed ticks after {warm}; "
                                       + ("unmodified reference (baseline/_ref, citywalk CrowdField.step)"
                                          if use_ref else "oracle port of the reference algorithm")
                                       + f"; wall {wall:.1f}s incl. scene sampling"},
            "e2e": {"value": round(v, 3), "unit": "env-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "scenes_per_sec": round(usable / t_scene, 4),
            "sample_includes": "generate_scene (zones, WFC terrain, placement, raster + heightfield, route "
                               "anchors), spawn_agents, CrowdField prep (nearest-obstacle map); one scene "
                               "per process"}
    print(json.dumps(line), flush=True)


def relaunch(args):
    """--gpus N without torchrun: re-exec this script under torch.distributed.run."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--envs", type=int, default=None)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="run", choices=["run", "step"],
                    help="value through CrowdField.run (default) or K CrowdField.step calls")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--threads", type=int, default=None)
    ap.add_argument("--sample-warmup", type=int, default=1)
    ap.add_argument("--sample-reps", type=int, default=3)
    ap.add_argument("--sync-steps", type=int, default=100)
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--cpu-steps", type=int, default=20)
    ap.add_argument("--ref-steps", type=int, default=500)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-step-batch", action="store_true")
    ap.add_argument("--no-standby", action="store_true",
                    help="cfg5 per-tick loops: re-sample at each reset instead of from the standby pool")
    ap.add_argument("--run-chunk", type=int, default=25,
                    help="ticks per CrowdField.run call in the run-mode e2e measurement")
    ap.add_argument("--phase-steps", type=int, default=50)
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per launch of the dominant kernel from an ncu --set full capture")
    args = ap.parse_args()
    CFG.clear()
    CFG.update(CONFIGS[args.config])
    if args.envs is None:
        args.envs = CFG["envs"]
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

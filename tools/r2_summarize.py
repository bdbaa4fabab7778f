"""Summaries under profiles/ from the round-2 ncu exports in gpurun_out/ (tools/r2_profile.sh):
  r2_ncu_step_<cfg>.txt + r2_traffic_<cfg>.json   synchronous-tick kernels, --set full
  r2_ncu_sampling_cfg2.txt                          sampling kernels, --set full
  r2_ncu_run_range_cfg2.txt                         the headline CrowdField.run as one app-range
  r2_launches_cfg2.txt                              launch list of the default bench command
"""
import csv
import io
import json
import os
import re
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r2"
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6, "second": 1e3}


def raw(path):
    rows = list(csv.reader(open(path)))
    rows = [r for r in rows if r and not r[0].startswith("==")]
    return rows[0], rows[1], rows[2:]


def short(name):
    m = re.search(r"(k_\w+(?:<[^>]*>)?)", name)
    return m.group(1) if m else name[:40]


def kernel_blocks(path, header):
    hdr, units, rows = raw(path)
    u = dict(zip(hdr, units))
    lines = [header, ""]
    recs = []
    for r in rows:
        d = dict(zip(hdr, r))
        lines.append("-" * 60)
        lines.append(f"  {'Kernel Name':62s} {d.get('Kernel Name', '')[:90]}")
        for k in WANT:
            if k in d:
                lines.append(f"  {k:62s} {d[k]} {u.get(k, '')}")
        recs.append((d, u))
    return lines, recs


def val(d, u, k):
    v = float(d[k].replace(",", ""))
    return v * SCALE.get(u[k], 1.0)


def main():
    os.makedirs(P, exist_ok=True)
    for cfg in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"):
        path = os.path.join(G, f"{TAG}_step_{cfg}_raw.csv")
        if not os.path.exists(path):
            continue
        hdr = (f"ncu --set full --clock-control none --import-source on --profile-from-start off "
               f"-k regex:'k_astar|k_orca|k_guide'\n  python tools/tick_once.py {cfg} 20   (the bench state after 20 "
               f"ticks, then one tick phase by phase: k_guide, k_astar, k_orca over all envs; cold, serialised)")
        lines, recs = kernel_blocks(path, hdr)
        open(os.path.join(P, f"{TAG}_ncu_step_{cfg}.txt"), "w").write("\n".join(lines) + "\n")
        kern = {}
        for d, u in recs:
            n = short(d["Kernel Name"]).split("<")[0]
            kern[n] = {"dram_read_bytes": val(d, u, "dram__bytes_read.sum"),
                       "dram_write_bytes": val(d, u, "dram__bytes_write.sum"),
                       "duration_ms": val(d, u, "gpu__time_duration.sum"),
                       "issue_active_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"])}
        json.dump({"source": f"ncu --set full --clock-control none (profiles/{TAG}_ncu_step_{cfg}.txt), {cfg} "
                             f"synchronous tick, one launch each", "kernels": kern},
                  open(os.path.join(P, f"{TAG}_traffic_{cfg}.json"), "w"), indent=1)
    path = os.path.join(G, f"{TAG}_sample_cfg2_raw.csv")
    if os.path.exists(path):
        lines, recs = kernel_blocks(path, "ncu --set full --clock-control none --import-source on "
                                          "-k regex:'k_zones|k_terrain|k_place|k_raster|k_footprint|k_nearest|"
                                          "k_walk|k_reach|k_spawn|k_routes|k_seeds' -c 16\n  python "
                                          "tools/sample_once.py cfg2   (1024 envs, 256^2)")
        tot = defaultdict(lambda: [0.0, 0.0, 0])
        for d, u in recs:
            n = short(d["Kernel Name"])
            t = tot[n]
            t[0] += val(d, u, "gpu__time_duration.sum")
            t[1] += val(d, u, "dram__bytes_read.sum") + val(d, u, "dram__bytes_write.sum")
            t[2] += 1
        s = sum(v[0] for v in tot.values())
        lines += ["", "per kernel (serialised, cold):  ms  share  dram MB  GB/s"]
        for n, (t, b, c) in sorted(tot.items(), key=lambda x: -x[1][0]):
            lines.append(f"  {n:24s} x{c}  {t:8.3f}  {t / s:5.3f}  {b / 1e6:8.1f}  {b / 1e9 / (t / 1e3):8.1f}")
        open(os.path.join(P, f"{TAG}_ncu_sampling_cfg2.txt"), "w").write("\n".join(lines) + "\n")
    path = os.path.join(G, f"{TAG}_run_range_cfg2_raw.csv")
    if os.path.exists(path):
        hdr, units, rows = raw(path)
        u = dict(zip(hdr, units))
        d = dict(zip(hdr, rows[0]))
        lines = ["CW_PROFILE_RANGE=1 ncu --replay-mode app-range --clock-control none --metrics ... \\",
                 "  python bench.py --steps 100 --warmup 20 ...   (cfg2)",
                 "range = the timed CrowdField.run(100) (cudaProfilerStart/Stop around it): every kernel of the",
                 "run -- persistent search server(s), round kernels, init/finish -- executing concurrently", ""]
        for k in hdr:
            if k.endswith(".sum") or k.endswith("pct_of_peak_sustained_active") or "elapsed" in k:
                if any(s in k for s in ("dram", "gpu__time", "inst_executed", "issue_active", "warps_active",
                                        "sm__throughput")):
                    lines.append(f"  {k:62s} {d[k]} {u[k]}")
        t = val(d, u, "gpu__time_duration.sum")
        b = val(d, u, "dram__bytes_read.sum") + val(d, u, "dram__bytes_write.sum")
        lines += ["", f"  range time {t:.3f} ms for 100 ticks ({t / 100:.4f} ms/tick under the profiler); "
                      f"DRAM {b / 1e6:.1f} MB = {b / 100 / 1e6:.2f} MB/tick, {b / 1e9 / (t / 1e3):.1f} GB/s"]
        open(os.path.join(P, f"{TAG}_ncu_run_range_cfg2.txt"), "w").write("\n".join(lines) + "\n")
    path = os.path.join(G, f"{TAG}_launches_cfg2.csv")
    if os.path.exists(path):
        rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
        hdr = rows[0]
        tot = defaultdict(lambda: [0.0, 0])
        for r in rows[1:]:
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            t = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
            n = short(d["Kernel Name"]) if "cw::" in d["Kernel Name"] else "torch/other"
            tot[n][0] += t
            tot[n][1] += 1
        s = sum(v[0] for v in tot.values())
        lines = ["ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv  python bench.py --steps 10 "
                 "--warmup 3 --no-cpu-baseline --no-step-batch --sample-reps 1 --sync-steps 2 --e2e-steps 2 "
                 "--phase-steps 2", "(default bench command shape, cfg2, run mode; per-launch times are cold and "
                 "serialised -- the run's kernels complete without running concurrently)", "",
                 f"{'kernel':40s} {'n':>5s} {'sum ms':>10s} {'avg us':>10s} {'share':>6s}"]
        for n, (t, c) in sorted(tot.items(), key=lambda x: -x[1][0]):
            lines.append(f"{n:40s} {c:5d} {t:10.3f} {1e3 * t / c:10.1f} {t / s:6.3f}")
        open(os.path.join(P, f"{TAG}_launches_cfg2.txt"), "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()

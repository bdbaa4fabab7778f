"""Drive the lane-per-agent ORCA body through synchronous phase launches so ncu can
capture it (the multi-tick run cannot run under kernel-serialising ncu).

  CW_ORCA_LANES=1 ncu --set full --clock-control none --import-source on \
      -k regex:k_orca -s 82 -c 1 -o gpurun_out/orca_lanes python tools/orca_lane_prof.py

Reuses tools/run_probe.py's setup (cfg2 by default, CFG=cfgN to change), then runs
guide / A* / ORCA as separate phases with 64-thread CTAs.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
src = open(os.path.join(HERE, "run_probe.py")).read()
src = src[:src.index("f, h = fields")]
sys.argv = ["run_probe.py", "10", os.environ.get("CFG", "cfg2")]
g = {"__file__": os.path.join(HERE, "run_probe.py"), "__name__": "run_probe_head"}
exec(compile(src, "run_probe_head", "exec"), g)
f, rpos, rvel, torch = g["fields"][0], g["rpos"], g["rvel"], g["torch"]
f.threads = 64
for _ in range(4):
    for ph in (1, 2, 4):
        f.step_phase(ph, rpos, rvel, 0.35)
torch.cuda.synchronize()

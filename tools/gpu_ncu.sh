#!/bin/bash
# ncu passes for the cfg2 step (run only after bench.py exited 0 without ncu).
# --no-run: ncu serialises kernels, and the multi-tick run's search server waits
# on round kernels running beside it, so only the synchronous tick is profiled.
#  1) launch list of a short bench (per-launch gpu__time_duration, cold / serialised)
#  2) one --set full capture of the top kernel (k_astar) with source
set -x
mkdir -p gpurun_out
TAG=${1:-r1}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline \
  --sample-reps 1 --e2e-steps 2 --phase-steps 2 --no-run > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_astar|k_orca|k_guide' -s 60 -c 3 \
  -o gpurun_out/${TAG}_step python bench.py --steps 30 --warmup 20 --no-cpu-baseline --sample-reps 1 \
  --e2e-steps 1 --phase-steps 1 --no-run > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done

#!/bin/bash
# Round-2 ncu evidence (run on the GPU box only after `python bench.py` exited 0 without ncu).
# Reports go to $NCU_DIR (not copied back); CSV exports land in gpurun_out/ (small):
#  1) launch list of the default bench command (run mode, per-launch gpu__time_duration;
#     cold and serialised -- the run no longer needs concurrent kernels, so it completes)
#  2) --set full of the synchronous tick's kernels (k_guide, k_astar, k_orca) per config
#  3) --set full of every sampling kernel at cfg2 (1024 envs)
#  4) the headline run as one ncu range (app-range replay): counters over the whole
#     CrowdField.run with its kernels running concurrently
mkdir -p gpurun_out
TAG=${TAG:-r2}
NCU_DIR=${NCU_DIR:-/tmp/ncu_$TAG}
mkdir -p $NCU_DIR
CFGS=${CFGS:-"cfg1 cfg2 cfg3 cfg4 cfg5"}
STEPS=${STEPS:-1}
SAMPLE=${SAMPLE:-1}
RANGE=${RANGE:-1}
LAUNCH=${LAUNCH:-1}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ "$LAUNCH" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches_cfg2.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline \
    --no-step-batch --sample-reps 1 --sync-steps 2 --e2e-steps 2 --phase-steps 2 \
    > gpurun_out/${TAG}_ncu_launch.log 2>&1
  echo "launch list rc=$?"
fi
if [ "$STEPS" = 1 ]; then
  for C in $CFGS; do
    timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
      -k regex:'k_astar|k_orca|k_guide' -o $NCU_DIR/step_${C} -f python tools/tick_once.py $C 20 \
      > gpurun_out/${TAG}_ncu_step_${C}.log 2>&1
    echo "step $C rc=$?"
    ncu -i $NCU_DIR/step_${C}.ncu-rep --page raw --csv > gpurun_out/${TAG}_step_${C}_raw.csv 2>/dev/null
  done
fi
if [ "$SAMPLE" = 1 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:'k_zones|k_terrain|k_place|k_raster|k_footprint|k_nearest|k_walk|k_reach|k_spawn|k_routes|k_seeds' \
    -c 16 -o $NCU_DIR/sample_cfg2 -f python tools/sample_once.py cfg2 > gpurun_out/${TAG}_ncu_sample.log 2>&1
  echo "sample rc=$?"
  ncu -i $NCU_DIR/sample_cfg2.ncu-rep --page raw --csv > gpurun_out/${TAG}_sample_cfg2_raw.csv 2>/dev/null
fi
if [ "$RANGE" = 1 ]; then
  CW_PROFILE_RANGE=1 timeout 1200 ncu --replay-mode app-range --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed \
    -o $NCU_DIR/run_range_cfg2 -f python bench.py --steps 100 --warmup 20 --no-cpu-baseline --no-step-batch \
    --sample-reps 1 --sync-steps 2 --e2e-steps 2 --phase-steps 2 > gpurun_out/${TAG}_ncu_range.log 2>&1
  echo "range rc=$?"
  ncu -i $NCU_DIR/run_range_cfg2.ncu-rep --page raw --csv > gpurun_out/${TAG}_run_range_cfg2_raw.csv 2>/dev/null
fi
du -sh gpurun_out

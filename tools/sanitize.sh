#!/bin/bash
# compute-sanitizer passes over small device workloads (GPU box).  Logs in gpurun_out/san/.
#   memcheck: parity tests (sampling + crowd), the drop-in entry points, the run (incl. the
#             relaunchable search server) and the routes; racecheck / synccheck: A* and ORCA tests.
mkdir -p gpurun_out/san
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
S="compute-sanitizer --error-exitcode 7 --print-limit 20"
run() { local name=$1; shift; timeout 1500 $S "$@" > gpurun_out/san/$name.log 2>&1; echo "rc=$?" >> gpurun_out/san/$name.log; }
run memcheck_parity --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not shard"
run memcheck_dropin --tool memcheck python -m pytest tests/test_gpu_dropin.py -m gpu -x -q
run memcheck_run --tool memcheck python -m pytest tests/test_gpu_run.py -m gpu -x -q -k "edge_cases or env_mask"
run memcheck_routes --tool memcheck python -m pytest tests/test_gpu_routes.py -m gpu -x -q
run racecheck_astar --tool racecheck python -m pytest tests/test_gpu_astar.py -m gpu -x -q -k "regress"
run synccheck_parity --tool synccheck python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "trajectory"
grep -H "rc=\|ERROR SUMMARY" gpurun_out/san/*.log

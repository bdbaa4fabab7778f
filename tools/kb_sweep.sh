#!/bin/bash
# run-mode server shared-memory budget sweep on the default bench (cfg2): value per budget
for rep in 1 2; do
  for kb in 220 200 190 180 170; do
    v=$(CW_RUN_SERVER_KB=$kb python bench.py --no-cpu-baseline --no-step-batch --sync-steps 5 --e2e-steps 5 \
        --phase-steps 5 --sample-reps 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])")
    echo "kb $kb: $v"
  done
done

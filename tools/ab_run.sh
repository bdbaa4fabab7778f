#!/bin/bash
# A/B two prebuilt libraries on the multi-tick run probe:
# tools/ab_run.sh <ticks> [config]   (tools/_ab/libA.so vs tools/_ab/libB.so, alternating)
T=${1:-500}
C=${2:-cfg2}
for v in A B A B A B; do
  cp tools/_ab/lib$v.so paper_2505_00690_b200/libcitywalk_b200.so
  touch paper_2505_00690_b200/libcitywalk_b200.so
  echo "lib$v: $(python tools/run_probe.py $T $C 2>&1 | tail -1)"
done

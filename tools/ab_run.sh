#!/bin/bash
# A/B two variant libraries on the multi-tick run probe, alternating, via CW_LIB_PATH:
#   tools/ab_run.sh <ticks> [config] [A.so] [B.so]   (build variants with tools/ab_build.sh)
T=${1:-500}
C=${2:-cfg2}
A=${3:-tools/_ab/A.so}
B=${4:-tools/_ab/B.so}
for v in "$A" "$B" "$A" "$B" "$A" "$B"; do
  echo "$(basename "$v"): $(CW_LIB_PATH="$v" python tools/run_probe.py "$T" "$C" 2>&1 | tail -1)"
done

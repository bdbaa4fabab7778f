#!/bin/bash
# A/B two variant libraries on the A* lab without touching the in-tree .so:
#   tools/ab.sh <ticks> <A.so> <B.so>   (build variants with tools/ab_build.sh)
T=${1:-8}
A=${2:-tools/_ab/A.so}
B=${3:-tools/_ab/B.so}
for v in "$A" "$B" "$A" "$B"; do
  echo "$(basename "$v"): $(CW_LIB_PATH="$v" python tools/astar_lab.py "$T" 20 2>&1 | tail -1)"
done

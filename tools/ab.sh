#!/bin/bash
# A/B two prebuilt libraries on the A* lab: tools/ab.sh <ticks> (libA = working tree, libB = HEAD)
T=${1:-8}
for v in A B A B; do
  cp tools/_ab/lib$v.so paper_2505_00690_b200/libcitywalk_b200.so
  touch paper_2505_00690_b200/libcitywalk_b200.so
  echo "lib$v: $(python tools/astar_lab.py $T 20 2>&1 | tail -1)"
done

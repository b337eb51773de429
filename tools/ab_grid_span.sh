#!/bin/bash
# In-graph device span (CUPTI, tools/timeline.py) of one-level solves with the
# grid kernel (TPB_GRID=1) and the level path (TPB_GRID=0), TPB_GRID_MIN=4.
for spec in "1e3 4" "3e3 4" "1e4 4" "1e4 8" "3e4 16" "6e4 20" "1e5 32" "2e5 32" "4e5 32" "6e5 32" "1e6 32"; do
  set -- $spec
  for g in 0 1; do
    s=$(TPB_GRID_MIN=4 TPB_GRID=$g python tools/timeline.py --n $1 --policy $2 2>/dev/null | grep span)
    echo "n=$1 m=$2 grid=$g $s"
  done
done

#!/bin/bash
# In-graph device span (CUPTI, tools/timeline.py) with the grid solve taking the
# deepest fitting level (TPB_GRID=1, default) vs the level path (TPB_GRID=0).
for spec in "1e8 64,10,32,16" "12499840 64,10,32,16" "1.25e7 64,10,32,16" "4e6 32,32" "1e7 32,10,32,8" "3e6 32,32" "2e6 32" "1e9 64,10,32,32"; do
  set -- $spec
  for g in 0 1; do
    for r in 1 2; do
      s=$(TPB_GRID=$g python tools/timeline.py --n $1 --policy $2 2>/dev/null | grep -E "span|grid_solve" | tr '\n' ' ')
      echo "n=$1 p=$2 grid=$g $s"
    done
  done
done

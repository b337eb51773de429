#!/bin/bash
# k_grid_hyb (TPB_GRID_HYB=1: rows via registers into shared memory) vs the default selection
# (k_grid_solve / k_grid_reg): in-graph grid-kernel duration (CUPTI), 3 runs each.
for spec in "1e5 32" "4e5 32" "6e5 32" "1e6 32" "6e5 20" "1e8 64,10,32,16" "12499840 64,10,32,16"; do
  set -- $spec
  for g in 0 1; do
    for r in 1 2 3; do
      d=$(TPB_GRID_HYB=$g python tools/timeline.py --n $1 --policy $2 2>/dev/null | grep -E "k_grid" | awk '{print $2}')
      echo "n=$1 p=$2 hyb=$g grid_kernel_us=$d"
    done
  done
done

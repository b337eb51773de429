#!/bin/bash
# A/B of the fused deepest level (TPB_FUSE_LAST) on the C1..C4 device solves
for rep in 1 2 3; do for f in 0 1; do
  for cfg in "1e4" "1e6" "1e8"; do
    TPB_FUSE_LAST=$f python tools/solve_time.py --n $cfg --tag "fuse=$f rep=$rep"
  done
done; done

#!/bin/bash
# A/B of the one-kernel grid solve (TPB_GRID) against the level path, for the
# one-level policies at small and mid N; phase traces and in-graph timelines of C1/C2.
export TPB_GRID_MIN=4
for spec in "1e4 4" "1e4 8" "3e4 16" "1e5 32" "3e5 32" "1e6 32" "1e6 16" "1e6 64"; do
  set -- $spec
  for g in 0 1; do TPB_GRID=$g python tools/solve_time.py --n $1 --policy $2 --steps 300 --tag grid=$g; done
done
TPB_GRID_TRACE=1 python tools/grid_trace.py --n 1e6 --policy 32 --out gpurun_out/grid_trace_c2.json
TPB_GRID_TRACE=1 python tools/grid_trace.py --n 1e4 --policy 4 --out gpurun_out/grid_trace_c1.json
python tools/timeline.py --n 1e6 --policy 32 --out gpurun_out/grid_timeline_c2.json > gpurun_out/grid_timeline_c2.txt 2>&1
python tools/timeline.py --n 1e4 --policy 4 --out gpurun_out/grid_timeline_c1.json > gpurun_out/grid_timeline_c1.txt 2>&1

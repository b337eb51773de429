#!/bin/bash
# In-graph (CUPTI) span A/B of library variants / env switches for one (N, policy):
#   tools/ab_timeline.sh "1e6" "32" "TPB_LIB=lib/variants/a.so" "TPB_LIB=lib/variants/b.so X=1" ...
# (back-to-back replays are host-bound below ~25 us, so solve_time.py cannot
# resolve the grid solve; the timeline tool measures the kernel itself)
n=$1; pol=$2; shift 2
for rep in 1 2 3; do for e in "$@"; do
  s=$(env $e python tools/timeline.py --n $n --policy $pol 2>/dev/null | grep '^span' | awk '{print $2}')
  echo "rep=$rep n=$n policy=$pol [$e] span_us=$s"
done; done

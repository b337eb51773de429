#!/bin/bash
# A/B of the single-GPU graph against the 1-rank fused sharded graph (same
# box, alternating, so power capping hits both arms alike).
# usage: tools/ab_sharded.sh [rounds] [extra bench args]
R=${1:-3}; shift
for i in $(seq 1 $R); do
  python bench.py --e2e-steps 0 --no-cpu-baseline "$@" | sed "s/^/single $i /"
  python bench.py --force-sharded --e2e-steps 0 --no-cpu-baseline "$@" | sed "s/^/shard_p2p $i /"
  python bench.py --force-sharded --transport nccl --e2e-steps 0 --no-cpu-baseline "$@" | sed "s/^/shard_nccl $i /"
done

#!/bin/bash
# A/B of env switches on device solves: tools/ab_env.sh "VAR=a" "VAR=b" -- N1 N2 ...
envs=(); while [ "$1" != "--" ] && [ -n "$1" ]; do envs+=("$1"); shift; done; shift
for rep in 1 2 3; do for e in "${envs[@]}"; do for n in "$@"; do
  env $e python tools/solve_time.py --n $n --tag "$e rep=$rep"
done; done; done

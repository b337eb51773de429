#!/bin/bash
# A/B of two library builds (TPB_LIB) on device solve time, alternating runs:
#   bash tools/ab_lib.sh OLD.so NEW.so "1e8 64" "2e6 32" ...
old=$1; new=$2; shift 2
for spec in "$@"; do
  set -- $spec
  for rep in 1 2 3; do
    for lib in "$old" "$new"; do
      TPB_LIB=$lib python tools/solve_time.py --n $1 ${2:+--policy $2} --steps 200 --tag "$(basename $lib)"
    done
  done
done

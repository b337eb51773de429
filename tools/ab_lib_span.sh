#!/bin/bash
# A/B of two library builds on in-graph spans (tools/timeline.py), alternating, 3 runs each:
#   bash tools/ab_lib_span.sh OLD.so NEW.so "1e4 4" "3e4 16" ...
old=$1; new=$2; shift 2
for spec in "$@"; do
  set -- $spec
  for rep in 1 2 3; do
    for lib in "$old" "$new"; do
      echo "$(basename $lib) n=$1 p=$2 $(TPB_LIB=$lib python tools/timeline.py --n $1 --policy $2 2>/dev/null | grep span)"
    done
  done
done

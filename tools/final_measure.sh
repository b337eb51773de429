#!/bin/bash
# round-end measurement set: tools/round_measure.sh + the four sanitizers over tools/sanitize_cases.py
bash tools/round_measure.sh > gpurun_out/rm.log 2>&1
for t in memcheck racecheck synccheck initcheck; do
  echo "== $t"; timeout 900 compute-sanitizer --tool $t python tools/sanitize_cases.py 2>&1 | grep -E "SUMMARY|sanitize cases" | head -3
done > gpurun_out/sanitizer.txt 2>&1
cat gpurun_out/sanitizer.txt

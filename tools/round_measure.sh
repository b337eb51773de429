#!/bin/bash
# end-of-change measurement (round $R, default r02): bench line, reference arm,
# launch list, ncu full captures of C3 / C2 / C1, in-graph timelines C1-C4,
# grid-kernel phase traces. Everything lands in gpurun_out/ (copy to profiles/).
# Under gpurun the three .ncu-rep files together exceed the 64 MiB copy-back
# cap: run tools/round_measure_small.sh and one ncu capture per call instead.
R=${R:-r02}
set -x
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_ref.json 2> gpurun_out/${R}_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 3 --prewarm 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${R}_ncu_bench.log 2>&1
K='regex:k_fast|k_generic|k_final|k_level_final|k_grid|k_split'
ncu --set full --clock-control none --import-source on -k "$K" -o gpurun_out/${R}_c3 -f python tools/ncu_capture.py > gpurun_out/${R}_capture_c3.log 2>&1
cp gpurun_out/ncu_labels.json gpurun_out/${R}_labels_c3.json
ncu --set full --clock-control none --import-source on -k "$K" -o gpurun_out/${R}_c2 -f python tools/ncu_capture.py --n 1e6 --policy 32 > gpurun_out/${R}_capture_c2.log 2>&1
cp gpurun_out/ncu_labels.json gpurun_out/${R}_labels_c2.json
ncu --set full --clock-control none --import-source on -k "$K" -o gpurun_out/${R}_c1 -f python tools/ncu_capture.py --n 1e4 --policy 4 > gpurun_out/${R}_capture_c1.log 2>&1
cp gpurun_out/ncu_labels.json gpurun_out/${R}_labels_c1.json
python tools/timeline.py --out gpurun_out/${R}_timeline_c3.json > gpurun_out/${R}_timeline_c3.txt 2>&1
python tools/timeline.py --n 1e6 --policy 32 --out gpurun_out/${R}_timeline_c2.json > gpurun_out/${R}_timeline_c2.txt 2>&1
python tools/timeline.py --n 1e9 --policy 64,10,32,32 --out gpurun_out/${R}_timeline_c4.json > gpurun_out/${R}_timeline_c4.txt 2>&1
python tools/timeline.py --n 1e4 --policy 4 --out gpurun_out/${R}_timeline_c1.json > gpurun_out/${R}_timeline_c1.txt 2>&1
# the stamps live only in a trace build: make -C paper_2510_27351_b200/csrc TRACE=1 OUT=../lib/trace
TPB_LIB=paper_2510_27351_b200/lib/trace/libtridpart_b200.so TPB_GRID_TRACE=1 python tools/grid_trace.py --n 1e6 --policy 32 --out gpurun_out/${R}_grid_trace_c2.json > gpurun_out/${R}_grid_trace_c2.txt 2>&1

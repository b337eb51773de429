#!/bin/bash
# the small half of tools/round_measure.sh (everything but the ncu full captures)
R=${R:-r02}
set -x
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_ref.json 2> gpurun_out/${R}_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 3 --prewarm 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${R}_ncu_bench.log 2>&1
python tools/timeline.py --out gpurun_out/${R}_timeline_c3.json > gpurun_out/${R}_timeline_c3.txt 2>&1
python tools/timeline.py --n 1e6 --policy 32 --out gpurun_out/${R}_timeline_c2.json > gpurun_out/${R}_timeline_c2.txt 2>&1
python tools/timeline.py --n 1e9 --policy 64,10,32,32 --out gpurun_out/${R}_timeline_c4.json > gpurun_out/${R}_timeline_c4.txt 2>&1
python tools/timeline.py --n 1e4 --policy 4 --out gpurun_out/${R}_timeline_c1.json > gpurun_out/${R}_timeline_c1.txt 2>&1
TPB_LIB=paper_2510_27351_b200/lib/trace/libtridpart_b200.so TPB_GRID_TRACE=1 python tools/grid_trace.py --n 1e6 --policy 32 --out gpurun_out/${R}_grid_trace_c2.json > gpurun_out/${R}_grid_trace_c2.txt 2>&1

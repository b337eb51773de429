#!/bin/bash
# end-of-change measurement: bench line, launch list, ncu full capture of one solve
set -x
python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/m_ref.json 2> gpurun_out/m_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/m_launches.csv python bench.py --steps 2 --warmup 3 --prewarm 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/m_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_fast|k_generic|k_final|k_level_final" -o gpurun_out/m_solve -f python tools/ncu_capture.py > gpurun_out/m_capture.log 2>&1
python tools/timeline.py --out gpurun_out/m_timeline_c3.json > gpurun_out/m_timeline_c3.txt 2>&1
python tools/timeline.py --n 1e6 --policy 32 --out gpurun_out/m_timeline_c2.json > gpurun_out/m_timeline_c2.txt 2>&1
python tools/timeline.py --n 1e9 --policy 64,10,32,32 --out gpurun_out/m_timeline_c4.json > gpurun_out/m_timeline_c4.txt 2>&1
python tools/timeline.py --n 1e4 --policy 8 --out gpurun_out/m_timeline_c1.json > gpurun_out/m_timeline_c1.txt 2>&1

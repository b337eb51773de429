# one-call measurement set (fits one gpurun call and the 64 MiB copy-back): GPU suite, smoke, bench, reference arm, timelines C1-C4 + the 8-GPU shard size, ncu C2 (summarised on the box), launch list, grid phase trace (needs the trace build)
R=${R:-r02s6}
K='regex:k_fast|k_generic|k_final|k_level_final|k_grid|k_split'
python -m pytest tests -m gpu -x -q > gpurun_out/${R}_gputest.log 2>&1; echo rc=$? >> gpurun_out/${R}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_ref.json 2> gpurun_out/${R}_ref.err
python tools/timeline.py --n 1e4 --policy 4 --out gpurun_out/${R}_timeline_c1.json > gpurun_out/${R}_timeline_c1.txt 2>&1
python tools/timeline.py --n 1e6 --policy 32 --out gpurun_out/${R}_timeline_c2.json > gpurun_out/${R}_timeline_c2.txt 2>&1
python tools/timeline.py --out gpurun_out/${R}_timeline_c3.json > gpurun_out/${R}_timeline_c3.txt 2>&1
python tools/timeline.py --n 1e9 --policy 64,10,32,32 --out gpurun_out/${R}_timeline_c4.json > gpurun_out/${R}_timeline_c4.txt 2>&1
python tools/timeline.py --n 12499840 --policy 64,10,32,16 > gpurun_out/${R}_timeline_shard.txt 2>&1
ncu --set full --clock-control none --import-source on -k "$K" -o gpurun_out/${R}_c2 -f python tools/ncu_capture.py --n 1e6 --policy 32 > gpurun_out/${R}_capture_c2.log 2>&1
python tools/ncu_capture.py --summarize gpurun_out/${R}_c2.ncu-rep --out gpurun_out/${R}_ncu_c2.json --md gpurun_out/${R}_ncu_full_summary_c2.md >> gpurun_out/${R}_capture_c2.log 2>&1
rm -f gpurun_out/${R}_c2.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 3 --prewarm 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/${R}_ncu_bench.log 2>&1
TPB_LIB=paper_2510_27351_b200/lib/trace/libtridpart_b200.so TPB_GRID_TRACE=1 python tools/grid_trace.py --n 1e6 --policy 32 --out gpurun_out/${R}_grid_trace_c2.json > gpurun_out/${R}_grid_trace_c2.txt 2>&1
tail -2 gpurun_out/${R}_gputest.log; cat gpurun_out/${R}_smoke.log; grep -h ^span gpurun_out/${R}_timeline_*.txt

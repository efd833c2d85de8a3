# Round evidence with the current code (one GPU): bench line, launch list, ncu full capture of
# the depth-0 kernels, shard scaling, report rows, progressive bench. Writes gpurun_out/ev_*.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ev_pytest.log 2>&1
python bench.py > gpurun_out/ev_bench_c4.json 2> gpurun_out/ev_bench_c4.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/ev_launches_c4.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_list.log 2>&1
python tools/launch_breakdown.py gpurun_out/ev_launches_c4.csv > gpurun_out/ev_launches_c4_summary.txt 2>&1
python tools/profile_run.py C4 --frames 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'wf_isect|wf_shade|wf_accumulate' -c 7 -o /tmp/ev_full python tools/profile_run.py C4 --frames 1 > gpurun_out/ev_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/ev_full.ncu-rep "# ncu --set full --clock-control none --import-source on, C4 chunk 0 (depth-0 scans, shade, accumulate, depth-1 closest scan); command: ncu --set full -k regex:'wf_isect|wf_shade|wf_accumulate' -c 7 python tools/profile_run.py C4 --frames 1" > gpurun_out/ev_ncu_c4_full.txt 2> gpurun_out/ev_ncu_traffic.json
ncu -i /tmp/ev_full.ncu-rep --page raw --csv > gpurun_out/ev_ncu_full_raw.csv
python tools/shard_scaling.py C4 > gpurun_out/ev_shard_scaling_c4.txt 2>&1
python tools/report_rows.py C2 C3 C4 C5 > gpurun_out/ev_report_rows.md 2> gpurun_out/ev_report_rows.err
python bench.py --mode progressive --steps 20 --warmup 3 > gpurun_out/ev_bench_c0_progressive.json 2> gpurun_out/ev_bench_c0.err

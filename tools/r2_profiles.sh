# round-2 profile captures (one GPU): bench launch list, c5 streaming kernels (ncu --set full),
# on-chip calibration of the lattice kernels (tools/onchip_calib.py). Run from the repo root.
set -x
python bench.py --steps 2 --warmup 3 --no-c5 --no-cpu-baseline > gpurun_out/lb_plain.json 2>gpurun_out/lb_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 2 --warmup 3 --no-c5 --no-cpu-baseline > gpurun_out/lb_ncu.log 2>&1
python tools/profile_eval.py c5 --solves 1 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"enum_count|window_select|frontier_bucket|frontier_items" -c 4 -o gpurun_out/r2_c5_streaming python tools/profile_eval.py c5 --solves 1 > gpurun_out/c5s.log 2>&1
python tools/onchip_calib.py run c2 > gpurun_out/calib_run.log 2>&1 && read SKIP COUNT < gpurun_out/calib_skip.txt && \
ncu --metrics smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.sum,sm__inst_executed_pipe_lsu.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:"lat_layer|lat_top_kernel" -s $SKIP -c $COUNT --log-file gpurun_out/calib_ncu.csv python tools/onchip_calib.py run c2 > gpurun_out/calib_ncu.log 2>&1
ls -la gpurun_out/

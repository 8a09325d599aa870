set -x
C5=1 timeout 900 python tools/quick_perf.py > gpurun_out/r3h_perf.jsonl 2>&1; cat gpurun_out/r3h_perf.jsonl
timeout 600 ncu --metrics smsp__inst_executed.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum --clock-control none -k regex:dgemm_abft -c 2 python tools/prof_target.py 8192 > gpurun_out/r3h_ncu.log 2>&1; grep -E "dgemm_abft|inst_executed|dmma|duration" gpurun_out/r3h_ncu.log
for f in tests/test_gpu_parity.py tests/test_gpu_encode_modes.py tests/test_gpu_intervals.py; do timeout 150 python -m pytest $f -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2; done

set -x
: > gpurun_out/r3g_timeline.jsonl
for cfg in "2048 2048 2048" "16384 16384 1024"; do
  for mode in ft; do
    timeout 120 python tools/dev_timeline.py $cfg $mode >> gpurun_out/r3g_timeline.jsonl 2>>gpurun_out/r3g_timeline.err
  done
done
cat gpurun_out/r3g_timeline.jsonl; tail -3 gpurun_out/r3g_timeline.err
C5=1 timeout 900 python tools/quick_perf.py > gpurun_out/r3g_perf.jsonl 2>&1; cat gpurun_out/r3g_perf.jsonl
timeout 300 python tools/dev_check_cost.py 8192 8192 32768 2048 > gpurun_out/r3g_check_cost.log 2>&1; cat gpurun_out/r3g_check_cost.log
for f in tests/test_gpu_intervals.py tests/test_gpu_parity.py tests/test_gpu_edge.py; do timeout 150 python -m pytest $f -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2; done

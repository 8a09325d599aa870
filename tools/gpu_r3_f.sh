set -x
C5=1 timeout 900 python tools/quick_perf.py > gpurun_out/r3f_perf.jsonl 2>&1; cat gpurun_out/r3f_perf.jsonl
: > gpurun_out/r3f_timeline.jsonl
for cfg in "2048 2048 2048" "16384 16384 1024" "8192 8192 8192"; do
  for mode in noft ft; do
    timeout 120 python tools/dev_timeline.py $cfg $mode >> gpurun_out/r3f_timeline.jsonl 2>>gpurun_out/r3f_timeline.err
  done
done
cat gpurun_out/r3f_timeline.jsonl; tail -3 gpurun_out/r3f_timeline.err

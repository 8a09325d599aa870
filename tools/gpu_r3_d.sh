# GPU tests file by file (short timeouts: the whole suite runs in ~2 min), then the timelines.
set -x
python -c "import oracle; oracle.build()"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()"; echo smoke_rc=$?
: > gpurun_out/r3d_pytest.log
for f in ${TESTS:-$(ls tests/test_gpu_*.py)}; do
  timeout ${PER_FILE_TIMEOUT:-150} python -m pytest $f -m gpu -q -x -p no:cacheprovider >> gpurun_out/r3d_pytest.log 2>&1
  echo "$f rc=$?" | tee -a gpurun_out/r3d_pytest.log
done
grep -E "passed|failed|rc=|Error|assert" gpurun_out/r3d_pytest.log | tail -40
: > gpurun_out/r3d_timeline.jsonl
for cfg in ${TL_CFGS:-"2048 2048 2048" "16384 16384 1024" "8192 8192 8192" "8192 8192 32768" "256 256 256"}; do
  for mode in noft ft; do
    timeout 120 python tools/dev_timeline.py $cfg $mode >> gpurun_out/r3d_timeline.jsonl 2>>gpurun_out/r3d_timeline.err
  done
done
cat gpurun_out/r3d_timeline.jsonl; tail -3 gpurun_out/r3d_timeline.err

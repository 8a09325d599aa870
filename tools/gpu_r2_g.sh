# reduce-scatter check pass: GPU tests, quick perf, dev check cost
set -x
python -c "import oracle; oracle.build()"
: > gpurun_out/r2i_pytest.log
for f in $(ls tests/test_gpu_*.py); do
  timeout 600 python -m pytest $f -m gpu -q -x -p no:cacheprovider >> gpurun_out/r2i_pytest.log 2>&1
  echo "$f rc=$?" | tee -a gpurun_out/r2i_pytest.log
done
grep -E "passed|failed|error" gpurun_out/r2i_pytest.log
timeout 600 python tools/quick_perf.py | tee gpurun_out/r2i_qp.jsonl
timeout 600 python tools/dev_check_cost.py 8192 8192 32768 2048 2>&1 | tail -3 | tee gpurun_out/r2i_check_cost.log
C5=1 SHAPES=32768x32768x32768NN timeout 600 python tools/quick_perf.py | tee -a gpurun_out/r2i_qp.jsonl

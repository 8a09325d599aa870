# few-wave k-split: GPU tests, quick perf, dev check cost, default bench line
set -x
python -c "import oracle; oracle.build()"
: > gpurun_out/r2m_pytest.log
for f in $(ls tests/test_gpu_*.py); do
  timeout 600 python -m pytest $f -m gpu -q -x -p no:cacheprovider >> gpurun_out/r2m_pytest.log 2>&1
  echo "$f rc=$?" | tee -a gpurun_out/r2m_pytest.log
done
grep -E "passed|failed|error" gpurun_out/r2m_pytest.log
timeout 600 python tools/quick_perf.py | tee gpurun_out/r2m_qp.jsonl
timeout 600 python tools/dev_check_cost.py 8192 8192 32768 2048 2>&1 | tail -2 | tee gpurun_out/r2m_check_cost.log
timeout 1500 python bench.py > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err; echo bench_rc=$?
tail -3 gpurun_out/r2m_bench.err

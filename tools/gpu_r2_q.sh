# GPU tests + default bench line (pool threshold, few-wave split test)
set -x
python -c "import oracle; oracle.build()"
: > gpurun_out/${TAG}_pytest.log
for f in $(ls tests/test_gpu_*.py); do
  timeout 600 python -m pytest $f -m gpu -q -x -p no:cacheprovider >> gpurun_out/${TAG}_pytest.log 2>&1
  echo "$f rc=$?" | tee -a gpurun_out/${TAG}_pytest.log
done
grep -E "passed|failed|error" gpurun_out/${TAG}_pytest.log
timeout 1500 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo bench_rc=$?
tail -3 gpurun_out/${TAG}_bench.err

# test + bench cycle: GPU tests file by file (own timeouts), the check-cost probe, then the
# default bench line.
set -x
python -c "import oracle; oracle.build()"
timeout 300 python tools/hang_probe.py > gpurun_out/r2_hang_probe.log 2>&1; echo probe_rc=$?
tail -3 gpurun_out/r2_hang_probe.log
timeout 300 python tools/dev_check_cost.py 8192 8192 32768 2048 > gpurun_out/r2_check_cost.log 2>&1; cat gpurun_out/r2_check_cost.log
: > gpurun_out/r2_pytest.log
for f in ${TESTS:-$(ls tests/test_gpu_*.py)}; do
  timeout ${PER_FILE_TIMEOUT:-600} python -m pytest $f -m gpu -q -x -p no:cacheprovider >> gpurun_out/r2_pytest.log 2>&1
  echo "$f rc=$?" | tee -a gpurun_out/r2_pytest.log
done
grep -E "passed|failed|rc=" gpurun_out/r2_pytest.log | tail -30
timeout 1200 python bench.py ${BENCH:---steps 5 --warmup 3} > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench_rc=$?
tail -3 gpurun_out/r2_bench.err

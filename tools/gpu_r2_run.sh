# round-2 evidence pass: GPU tests file by file (each under its own timeout, so a hang costs
# minutes, not the whole call), then optionally a bench run.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import oracle; oracle.build()"
timeout 300 python tools/hang_probe.py > gpurun_out/r2_hang_probe.log 2>&1; echo probe_rc=$?
cat gpurun_out/r2_hang_probe.log | tail -20
TESTS=${TESTS:-$(ls tests/test_*.py)}
: > gpurun_out/r2_pytest.log
for f in $TESTS; do
  timeout ${PER_FILE_TIMEOUT:-600} python -m pytest $f -m gpu -q -p no:cacheprovider >> gpurun_out/r2_pytest.log 2>&1
  echo "$f rc=$?" | tee -a gpurun_out/r2_pytest.log
done
grep -E "passed|failed|error|rc=" gpurun_out/r2_pytest.log | tail -40
if [ -n "$BENCH" ]; then
  timeout 900 python bench.py $BENCH > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo bench_rc=$?
  tail -c 2500 gpurun_out/r2_bench.json; tail -5 gpurun_out/r2_bench.err
fi

set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import oracle; oracle.build()"
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/r2_pytest1.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/r2_pytest1.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo bench_rc=$?
tail -c 3000 gpurun_out/r2_bench1.json; tail -20 gpurun_out/r2_bench1.err

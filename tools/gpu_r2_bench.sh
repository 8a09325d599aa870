# round-2 bench pass: the default line (with per-config lines and the interval sweep), then the
# overhead breakdown of the protected kernel at C5 (dev build: mode 32 = unprotected kernel on
# the 127-row grid of C^f).
set -x
python -c "import oracle; oracle.build()"
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench_full.json 2> gpurun_out/r2_bench_full.err; echo bench_rc=$?
tail -c 4000 gpurun_out/r2_bench_full.json; tail -5 gpurun_out/r2_bench_full.err
N=32768 timeout 600 python tools/exp_modes.py 0 32 > gpurun_out/r2_modes.log 2>&1; echo modes_rc=$?
cat gpurun_out/r2_modes.log

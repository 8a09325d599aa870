#!/bin/bash
# Round evidence: tests, smoke, default bench (C5), reference arm, per-config bench lines,
# ncu launch list of the bench command, ncu --set full of one noft + one FT launch at C5.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || true
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench rc=$?"; cat gpurun_out/bench_c5.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
for c in C2 C3 C4a C4b; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1; echo "ncu-list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dgemm_abft -c 2 -o gpurun_out/ncu_full_c5 \
  python tools/prof_target.py 32768 > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"; tail -2 gpurun_out/ncu_full.log
ls -la gpurun_out

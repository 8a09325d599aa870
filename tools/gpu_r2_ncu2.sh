set -x
timeout 300 python tools/dev_check_cost.py 8192 8192 32768 2048 > gpurun_out/r2_check_cost.log 2>&1; echo cc_rc=$?
cat gpurun_out/r2_check_cost.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'dgemm_abft|scale_kernel|block_sum|verify|row_check|axpby' --csv --log-file gpurun_out/r2_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-per-config --no-cpu-baseline --no-sweep > gpurun_out/r2_ncu_bench.log 2>&1; echo launches_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dgemm_abft -c 1 -o gpurun_out/r2_ncu_full_check python tools/prof_check.py 4096 4096 8192 512 > gpurun_out/r2_ncu_full_check.log 2>&1; echo ncu_full_rc=$?

# round-2 evidence on the committed build: ncu launch list of the bench (product kernels), metric
# passes of the protected / unprotected C5 launch (traffic, DMMA activity), a full capture of
# the protected kernel at 8192^3 and one with Kc = 512, the check-cost probe.
set -x
timeout 300 python tools/dev_check_cost.py 8192 8192 32768 2048 > gpurun_out/r2e_check_cost.log 2>&1; cat gpurun_out/r2e_check_cost.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'dgemm_abft|scale_kernel|block_sum|verify|row_check|axpby|dgemv' --csv --log-file gpurun_out/r2e_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-per-config --no-cpu-baseline > gpurun_out/r2e_ncu_bench.log 2>&1; echo launches_rc=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,lts__t_sector_hit_rate.pct,launch__registers_per_thread,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second
timeout 900 ncu --metrics $M --clock-control none -k regex:dgemm_abft -s 1 -c 1 -o gpurun_out/r2e_ncu_c5_ft python tools/prof_target.py 32768 > gpurun_out/r2e_ncu_c5_ft.log 2>&1; echo ncu_ft_rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:dgemm_abft -c 1 -o gpurun_out/r2e_ncu_c5_noft python tools/prof_target.py 32768 > gpurun_out/r2e_ncu_c5_noft.log 2>&1; echo ncu_noft_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dgemm_abft -c 2 -o gpurun_out/r2e_ncu_full_8192 python tools/prof_target.py 8192 > gpurun_out/r2e_ncu_full_8192.log 2>&1; echo ncu_full_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dgemm_abft -c 1 -o gpurun_out/r2e_ncu_full_check python tools/prof_check.py 4096 4096 8192 512 > gpurun_out/r2e_ncu_full_check.log 2>&1; echo ncu_full2_rc=$?

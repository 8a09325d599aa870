# round-2 (session 2) evidence: the default bench line, then the ncu launch list of a short bench
# run and metric passes of the protected / unprotected kernel at C5, and a full capture at 8192^3.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import oracle; oracle.build()"
timeout 1500 python bench.py > gpurun_out/r3e_bench.json 2> gpurun_out/r3e_bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/r3e_bench.json; tail -3 gpurun_out/r3e_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3e_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-per-config --no-cpu-baseline --no-sweep > gpurun_out/r3e_ncu_bench.log 2>&1; echo launches_rc=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,lts__t_sector_hit_rate.pct,launch__registers_per_thread,smsp__inst_executed.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:dgemm_abft -s 1 -c 1 -o gpurun_out/r3e_ncu_c5_ft python tools/prof_target.py 32768 > gpurun_out/r3e_ncu_c5_ft.log 2>&1; echo ncu_ft_rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:dgemm_abft -c 1 -o gpurun_out/r3e_ncu_c5_noft python tools/prof_target.py 32768 > gpurun_out/r3e_ncu_c5_noft.log 2>&1; echo ncu_noft_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dgemm_abft -c 2 -o gpurun_out/r3e_ncu_full_8192 python tools/prof_target.py 8192 > gpurun_out/r3e_ncu_full_8192.log 2>&1; echo ncu_full_rc=$?
ls -la gpurun_out/ | tail -20

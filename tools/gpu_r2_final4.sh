# round-2 final evidence (fourth pass: + generalized splits, device-written report, encoder-head CTAs, checked-build fixes)
# the default bench line (what the driver runs), the reference arm, the ncu launch list of the
# bench and metric passes of the protected / unprotected C5 launch.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import oracle; oracle.build()"
: > gpurun_out/r2zzz_pytest.log
for f in $(ls tests/test_*.py); do
  timeout ${PER_FILE_TIMEOUT:-600} python -m pytest $f -m gpu -q -p no:cacheprovider >> gpurun_out/r2zzz_pytest.log 2>&1
  echo "$f rc=$?" | tee -a gpurun_out/r2zzz_pytest.log
done
grep -E "passed|failed|error|rc=" gpurun_out/r2zzz_pytest.log | tail -40
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2zzz_smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python bench.py > gpurun_out/r2zzz_bench.json 2> gpurun_out/r2zzz_bench.err; echo bench_rc=$?
tail -c 3000 gpurun_out/r2zzz_bench.json; tail -5 gpurun_out/r2zzz_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2zzz_ref.json 2> gpurun_out/r2zzz_ref.err; echo ref_rc=$?
tail -c 1500 gpurun_out/r2zzz_ref.json
[ -n "$NO_NCU" ] && exit 0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'dgemm_abft|scale_kernel|block_sum|verify|row_check|axpby|dgemv' --csv --log-file gpurun_out/r2zzz_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-per-config --no-cpu-baseline > gpurun_out/r2zzz_ncu_bench.log 2>&1; echo launches_rc=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,lts__t_sector_hit_rate.pct,launch__registers_per_thread,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second
timeout 900 ncu --metrics $M --clock-control none -k regex:dgemm_abft -s 1 -c 1 -o gpurun_out/r2zzz_ncu_c5_ft python tools/prof_target.py 32768 > gpurun_out/r2zzz_ncu_c5_ft.log 2>&1; echo ncu_ft_rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:dgemm_abft -c 1 -o gpurun_out/r2zzz_ncu_c5_noft python tools/prof_target.py 32768 > gpurun_out/r2zzz_ncu_c5_noft.log 2>&1; echo ncu_noft_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:dgemm_abft -c 2 -o gpurun_out/r2zzz_ncu_full_8192 python tools/prof_target.py 8192 > gpurun_out/r2zzz_ncu_full_8192.log 2>&1; echo ncu_full_rc=$?

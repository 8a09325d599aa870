#!/bin/bash
python tools/prof_target.py 4096 > gpurun_out/prof_plain.log 2>&1 && \
FTBLAS_DEV_CS=1 ncu --set full --clock-control none --import-source on -k regex:dgemm_abft -c 2 -o gpurun_out/prof_m1 python tools/prof_target.py 4096 > gpurun_out/ncu_m1.log 2>&1
echo "ncu rc=$?"; tail -1 gpurun_out/ncu_m1.log

#!/bin/bash
python tools/prof_target.py 2048 > gpurun_out/prof_plain.log 2>&1 && \
FTBLAS_DEV_CS=2 ncu --set full --clock-control none --import-source on -k regex:dgemm_abft -s 1 -c 1 -o gpurun_out/prof_m2 python tools/prof_target.py 2048 > gpurun_out/ncu_m2.log 2>&1
echo "ncu rc=$?"; tail -1 gpurun_out/ncu_m2.log

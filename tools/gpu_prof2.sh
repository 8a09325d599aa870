#!/bin/bash
python tools/prof_target.py 4096 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dgemm_abft -c 2 -o gpurun_out/prof_v2 python tools/prof_target.py 4096 > gpurun_out/ncu_v2.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_v2.log

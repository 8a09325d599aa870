#!/bin/bash
./microbench/fp64_interleave > gpurun_out/interleave.json 2>&1; cat gpurun_out/interleave.json
python tools/prof_target.py 4096 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dgemm_abft -c 2 -o gpurun_out/prof_v1 python tools/prof_target.py 4096 > gpurun_out/ncu_v1.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_v1.log

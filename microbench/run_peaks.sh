#!/bin/bash
# Runs the FP64 ceiling microbenchmarks with nvidia-smi clock sampling.
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./microbench/fp64_peak > gpurun_out/fp64_peak.json 2>&1
python microbench/cublas_dgemm.py > gpurun_out/cublas_dgemm.json 2>&1
kill $SMI
nvidia-smi -q -d CLOCK,POWER > gpurun_out/smi_q.txt 2>&1
cat gpurun_out/fp64_peak.json gpurun_out/cublas_dgemm.json

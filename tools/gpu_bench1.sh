#!/bin/bash
python bench.py --config C5 --size 8192 --steps 2 --warmup 1 > gpurun_out/bench_8192.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/bench_8192.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/bench_ref.log
nproc; free -g | head -2
timeout 900 python bench.py > gpurun_out/bench_c5.log 2>&1; echo "rc=$?"; tail -5 gpurun_out/bench_c5.log

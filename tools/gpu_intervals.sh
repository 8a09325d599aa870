#!/bin/bash
# Interval (NEXT-1) cost: C5 and C4b at several Kc, fused encode, no e2e / cpu baseline.
for kc in 0 8192 4096 2048; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-unfused --interval $kc > gpurun_out/int_c5_$kc.json 2>&1; echo "C5 Kc=$kc rc=$?"
done
for kc in 0 8192 4096 2048 1024; do
  timeout 600 python bench.py --config C4b --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-unfused --interval $kc > gpurun_out/int_c4b_$kc.json 2>&1; echo "C4b Kc=$kc rc=$?"
done
for f in gpurun_out/int_*.json; do python -c "
import json,sys; d=json.load(open('$f')); a=d['abft']; print('$f', d['config']['interval_Kc'], round(a['tflops_protected'],2), 'ovh', round(a['overhead_pct'],2), 'units', a['units_checked'], 'det', a['detected'], a['corrected'], a['recomputed'])"; done

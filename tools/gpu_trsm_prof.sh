#!/bin/bash
# FT-DTRSM profile at 8192^2: launch list (unprotected + protected solve) and one full capture
# of the diagonal-block leaf kernel.
python tools/prof_trsm.py 8192 > gpurun_out/prof_trsm.log 2>&1 || { echo "prof_trsm failed"; tail gpurun_out/prof_trsm.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_trsm.csv \
  python tools/prof_trsm.py 8192 > gpurun_out/ncu_trsm.log 2>&1; echo "ncu-list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsm_leaf -s 2 -c 1 -o gpurun_out/ncu_leaf \
  python tools/prof_trsm.py 8192 > gpurun_out/ncu_leaf.log 2>&1; echo "ncu-leaf rc=$?"

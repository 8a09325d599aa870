#!/bin/bash
for m in 0 1 2 3; do echo "mode $m"; FTBLAS_DEV_CS=$m timeout 300 python tools/quick_perf.py 2>&1 | head -2; done

#!/bin/bash
# GPU pass after an encode change: build, smoke, gpu tests, encoder timing, quick perf
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python tools/dev_prof.py 4096
timeout 600 python tools/quick_perf.py > gpurun_out/quick_perf.log 2>&1; echo "perf rc=$?"; cat gpurun_out/quick_perf.log

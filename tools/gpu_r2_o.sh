# GPU tests + quick perf + C4a timeline (first-stage wait)
set -x
python -c "import oracle; oracle.build()"
: > gpurun_out/${TAG}_pytest.log
for f in $(ls tests/test_gpu_*.py); do
  timeout 600 python -m pytest $f -m gpu -q -x -p no:cacheprovider >> gpurun_out/${TAG}_pytest.log 2>&1
  echo "$f rc=$?" | tee -a gpurun_out/${TAG}_pytest.log
done
grep -E "passed|failed|error" gpurun_out/${TAG}_pytest.log
SHAPES=16384x16384x1024NN,8192x8192x8192NN,2048x2048x2048NN timeout 600 python tools/quick_perf.py | tee gpurun_out/${TAG}_qp.jsonl
timeout 300 python tools/dev_timeline.py 16384 16384 1024 2>&1 | grep "^{" | tee gpurun_out/${TAG}_tl.jsonl
timeout 300 python tools/dev_timeline.py 8192 8192 8192 2>&1 | grep "^{" | tee -a gpurun_out/${TAG}_tl.jsonl

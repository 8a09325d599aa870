# encoder-head CTAs: GPU tests, quick perf, 2048^3 grid timeline
set -x
python -c "import oracle; oracle.build()"
: > gpurun_out/${TAG}_pytest.log
for f in $(ls tests/test_gpu_*.py); do
  timeout 600 python -m pytest $f -m gpu -q -x -p no:cacheprovider >> gpurun_out/${TAG}_pytest.log 2>&1
  echo "$f rc=$?" | tee -a gpurun_out/${TAG}_pytest.log
done
grep -E "passed|failed|error" gpurun_out/${TAG}_pytest.log
timeout 900 python tools/quick_perf.py | tee gpurun_out/${TAG}_qp.jsonl
BETA=0.5 SHAPES=2048x2048x2048NN,4096x4096x2048NN,1024x1024x1024NN,1536x1536x1536NN timeout 300 python tools/quick_perf.py | tee -a gpurun_out/${TAG}_qp.jsonl
timeout 300 python tools/dev_timeline.py 2048 2048 2048 2>&1 | grep "^{" | tee gpurun_out/${TAG}_tl.jsonl

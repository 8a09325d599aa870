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
SHAPES=16384x512x16384NN,16384x516x16384NN,32768x32768x8192NN timeout 300 python tools/quick_perf.py | tee -a gpurun_out/${TAG}_qp.jsonl
TL_DUMP=gpurun_out/${TAG}_tl_c4b.npy timeout 300 python tools/dev_timeline.py 16384 512 16384 2>&1 | grep "^{" | tee gpurun_out/${TAG}_tl.jsonl

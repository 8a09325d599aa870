# quick perf incl. C5 and small shapes (noft codegen check), GPU tests
set -x
timeout 900 python tools/quick_perf.py | tee gpurun_out/${TAG}_qp.jsonl
C5=1 SHAPES=256x256x256NN,32768x32768x32768NN timeout 600 python tools/quick_perf.py | tee -a gpurun_out/${TAG}_qp.jsonl
python -c "import oracle; oracle.build()"
: > gpurun_out/${TAG}_pytest.log
for f in $(ls tests/test_gpu_*.py); do
  timeout 600 python -m pytest $f -m gpu -q -x -p no:cacheprovider >> gpurun_out/${TAG}_pytest.log 2>&1
  echo "$f rc=$?" | tee -a gpurun_out/${TAG}_pytest.log
done
grep -E "passed|failed|error" gpurun_out/${TAG}_pytest.log

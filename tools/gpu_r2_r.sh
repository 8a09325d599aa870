# GPU tests + quick perf (incl. 256^3) + host-cost loop (C1 call with report)
set -x
python -c "import oracle; oracle.build()"
: > gpurun_out/${TAG}_pytest.log
for f in $(ls tests/test_gpu_*.py); do
  timeout 600 python -m pytest $f -m gpu -q -x -p no:cacheprovider >> gpurun_out/${TAG}_pytest.log 2>&1
  echo "$f rc=$?" | tee -a gpurun_out/${TAG}_pytest.log
done
grep -E "passed|failed|error" gpurun_out/${TAG}_pytest.log
timeout 600 python tools/quick_perf.py | tee gpurun_out/${TAG}_qp.jsonl
SHAPES=256x256x256NN,512x512x512NN,1024x1024x1024NN,1536x1536x1536NN,1024x1024x4096NN timeout 300 python tools/quick_perf.py | tee -a gpurun_out/${TAG}_qp.jsonl
timeout 300 bash tools/host_cost.sh 2>&1 | tee gpurun_out/${TAG}_host_cost.log

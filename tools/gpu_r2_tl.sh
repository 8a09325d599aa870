# timeline build: per-tile phases and the grid-level view (span, busy fraction, wave starts)
set -x
for a in "2048 2048 2048" "2048 2048 2048 noft" "16384 16384 1024" "16384 16384 1024 noft" "8192 8192 8192"; do
  timeout 300 python tools/dev_timeline.py $a 2>&1 | grep "^{" | tee -a gpurun_out/r2_tl.jsonl
done

# timeline build: per-tile phases of the four trans combinations at 8192^3 (FT and noft)
for tr in NN NT TN TT; do
  timeout 300 python tools/dev_timeline.py 8192 8192 8192 ft $tr 2>&1 | grep '"mode"' | tee -a gpurun_out/r2t_tl.jsonl
  timeout 300 python tools/dev_timeline.py 8192 8192 8192 noft $tr 2>&1 | grep '"mode"' | tee -a gpurun_out/r2t_tl.jsonl
done

out=gpurun_out/tnsw; mkdir -p $out
for n in 2 3 4 8 12 16 24 32 48; do
for t in 128 192 256; do
  echo "[WS_TN=$t]" $(env ALPA_WS_TN=$t timeout 120 python tools/sweep_point.py $n 10 2>&1 | tail -1) | tee -a $out/summary.txt
done; done

out=gpurun_out/tnab; mkdir -p $out
for n in 16 64 11; do
for v in "" "ALPA_WS_TN=192" "ALPA_WS_TN=192 ALPA_MK_TN=192,128,192,128,192,192" "ALPA_WS_TN=128" "ALPA_MK_TN=192,128,256,128,256,256"; do
  echo "[$v]" $(env $v timeout 120 python tools/sweep_point.py $n 10 2>&1 | tail -1) | tee -a $out/summary.txt
done; done

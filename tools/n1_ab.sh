out=gpurun_out/n1; mkdir -p $out
for v in "" "ALPA_MK_SPLITS=1,4,1,4,1,4" "ALPA_MK_SPLITS=1,2,1,4,1,4" "ALPA_MK_SPLITS=1,4,1,4,1,4 ALPA_MK_TN=32,32,64,64,64,64" "ALPA_MK_TN=32,32,64,64,64,64"; do
  env $v timeout 120 python tools/sweep_point.py 1 10 2>&1 | tail -1 | tee -a $out/summary.txt
done
env ALPA_MK_SPLITS=1,4,1,4,1,4 timeout 120 python tools/sweep_point.py 6 10 2>&1 | tail -1 | tee -a $out/summary.txt

# A/B of the per-op token tiles of the persistent kernel (ALPA_MK_TN = qkv,o,mlp1,mlp2,enc1,enc2)
out=gpurun_out/ab_tn; mkdir -p $out
for v in 64,64,192,192,192,192 128,64,192,192,192,192 128,128,192,192,192,192 96,64,192,192,192,192 64,128,192,192,192,192; do
  ALPA_MK_TN=$v timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/b.json 2>/dev/null
  python -c "import json;d=json.load(open('$out/b.json'));print('TN=$v', round(d['ms_per_step'],3))" | tee -a $out/summary.txt
done
ALPA_MK_TN=128,64,192,192,192,192 ALPA_MK_TRACE=1 timeout 120 python tools/mk_trace.py --blocks 4 > $out/trace_q128.txt 2>&1

#!/bin/bash
# A/B of an environment knob: tools/mk_env_ab.sh tag VAR v1 v2 ...  (trace + bench per value)
tag=$1; var=$2; shift 2
out=gpurun_out/$tag
mkdir -p $out
i=0
for v in "$@"; do
  env $var=$v ALPA_MK_TRACE=1 timeout 120 python tools/mk_trace.py --blocks 4 > $out/trace_$i.txt 2>&1
  env $var=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench_$i.json 2>/dev/null
  echo "$i $v" >> $out/index.txt
  i=$((i+1))
done
echo done

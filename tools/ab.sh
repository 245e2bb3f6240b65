#!/bin/bash
# Generic A/B on the GPU box: bash tools/ab.sh <tag> "<env assignments>" ["<env assignments>" ...]
# Each config: bench ms/scene (+ a 4-block trace with --trace).
tag=$1; shift
out=gpurun_out/$tag; mkdir -p $out
i=0
for cfg in "$@"; do
  env $cfg timeout 150 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/b$i.json 2> $out/b$i.err
  python -c "import json;d=json.load(open('$out/b$i.json'));print('[$cfg]', round(d['ms_per_step'],3))" 2>&1 | tee -a $out/summary.txt
  env $cfg ALPA_MK_TRACE=1 timeout 120 python tools/mk_trace.py --blocks 4 --extra > $out/trace$i.txt 2>&1
  i=$((i+1))
done

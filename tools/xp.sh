#!/bin/bash
# Env-knob experiments on the GPU box: tools/xp.sh tag "ENV=.. ENV2=.." "ENV=.." ...
# (one bench per setting, --no-sweeps; trace of the first 4 blocks per setting)
tag=$1; shift
out=gpurun_out/$tag
mkdir -p $out
i=0
for setting in "$@"; do
  env $setting ALPA_MK_TRACE=1 timeout 120 python tools/mk_trace.py --blocks 4 --extra --dump $out/trace_$i.npz > $out/trace_$i.txt 2>&1
  env $setting timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-sweeps > $out/bench_$i.json 2> $out/bench_$i.err
  ms=$(python -c "import json;print(json.load(open('$out/bench_$i.json'))['ms_per_step'])" 2>/dev/null)
  echo "$i [$setting] ms/scene $ms" | tee -a $out/index.txt
  i=$((i+1))
done

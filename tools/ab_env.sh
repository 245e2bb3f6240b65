#!/bin/bash
# A/B of an environment knob (bench only, interleaved): tools/ab_env.sh tag rounds VAR v1 v2 ...
tag=$1; rounds=$2; var=$3; shift 3
out=gpurun_out/$tag
mkdir -p $out
for r in $(seq 1 $rounds); do
  for v in "$@"; do
    env $var=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/${v}_$r.json 2>/dev/null
    python -c "import json;d=json.load(open('$out/${v}_$r.json'));print('$var=$v', round(d['ms_per_step'],3))" | tee -a $out/summary.txt
  done
done

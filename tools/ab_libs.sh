#!/bin/bash
# A/B of library builds on one box: tools/ab_libs.sh tag rounds lib1.so lib2.so ...
# (interleaved bench runs, ms/scene per run)
tag=$1; rounds=$2; shift 2
out=gpurun_out/$tag
mkdir -p $out
for r in $(seq 1 $rounds); do
  for lib in "$@"; do
    n=$(basename $lib .so)
    ALPA_LIB=$PWD/$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/${n}_$r.json 2>/dev/null
    python -c "import json;d=json.load(open('$out/${n}_$r.json'));print('$n', round(d['ms_per_step'],3))" | tee -a $out/summary.txt
  done
done

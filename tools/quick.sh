#!/bin/bash
# Dev loop on the GPU box: tools/quick.sh tag [extra command]  (trace + bench)
tag=$1; shift
out=gpurun_out/$tag
mkdir -p $out
ALPA_MK_TRACE=1 timeout 120 python tools/mk_trace.py --blocks 4 --extra --dump $out/trace.npz > $out/trace.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err
if [ $# -gt 0 ]; then timeout 300 bash -c "$*" > $out/extra.txt 2>&1; fi
python -c "import json;d=json.load(open('$out/bench.json'));print('ms/scene', d['ms_per_step'])" | tee $out/ms.txt

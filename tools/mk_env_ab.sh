#!/bin/bash
# A/B of an environment knob of the persistent kernel: tools/mk_env_ab.sh tag VAR v1 v2 ...
tag=$1; var=$2; shift 2
out=gpurun_out/$tag
mkdir -p $out
for v in "$@"; do
  env $var=$v ALPA_MK_TRACE=1 timeout 120 python tools/mk_trace.py --blocks 4 > $out/trace_$v.txt 2>&1
done
echo done

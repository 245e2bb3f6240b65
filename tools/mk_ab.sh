#!/bin/bash
# A/B of persistent-kernel knobs: trace per ALPA_MK_FLAGS setting
tag=${1:-ab}
shift
out=gpurun_out/$tag
mkdir -p $out
for f in "$@"; do
  ALPA_MK=1 ALPA_MK_FLAGS=$f ALPA_MK_TRACE=1 timeout 120 python tools/mk_trace.py --blocks 4 > $out/trace_f$f.txt 2>&1
done
echo done

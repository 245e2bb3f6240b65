#!/bin/bash
tag=${1:-mk2}
out=gpurun_out/$tag
mkdir -p $out
ALPA_MK=1 ALPA_MK_TRACE=1 timeout 120 python tools/mk_trace.py --blocks 4 > $out/trace.txt 2>&1
ALPA_MK=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err
ALPA_MK=1 timeout 600 python -m pytest tests -q -m gpu -x > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
echo done

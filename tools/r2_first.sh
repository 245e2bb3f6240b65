#!/bin/bash
# round-2 first GPU session: full gpu suite, bench, trace
tag=${1:-r2a}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
timeout 1200 python -m pytest tests -q -m gpu -rA -s > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err
ALPA_MK_TRACE=1 timeout 120 python tools/mk_trace.py --blocks 4 > $out/mk_trace.txt 2>&1
echo done

#!/bin/bash
# dev session: persistent-kernel correctness + timing (on the GPU box)
tag=${1:-mk1}
out=gpurun_out/$tag
mkdir -p $out
timeout 120 python tools/run_iteration.py --blocks 2 --iters 2 > $out/smoke_mk.log 2>&1; echo "rc=$?" >> $out/smoke_mk.log
timeout 600 python -m pytest tests -q -m gpu -x > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench.json 2> $out/bench.err
ALPA_MK=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $out/bench_old.json 2> $out/bench_old.err
echo done

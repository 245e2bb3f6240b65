#!/bin/bash
# Round-2 evidence: GPU tests, smoke, bench (both arms), launch list, ncu full of the iteration kernel, trace
tag=${1:-r2final}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
timeout 1200 python -m pytest tests -q -m gpu -s > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $out/bench.json 2> $out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
ALPA_MK_TRACE=1 timeout 120 python tools/mk_trace.py --blocks 4 > $out/mk_trace.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'iter_kernel|rollout' -c 40 --csv \
    --log-file $out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sweeps > $out/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:iter_kernel -s 0 -c 1 \
    -o $out/iter_kernel python tools/run_iteration.py --blocks 36 --iters 1 --eager > $out/ncu_full.log 2>&1
echo done

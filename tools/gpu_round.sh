#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), launch list + ncu captures.
# Usage (on the box): bash tools/gpu_round.sh <tag>
tag=${1:-r1}
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/gpu.txt
timeout 600 python -m pytest tests -q -m gpu -x > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
# launch list of one graph-replayed bench run (kernels of ~1 iteration after warm-up)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2600 -c 300 --csv \
    --log-file $out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $out/ncu_launch.log 2>&1
# full captures of the dominant kernels
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:tc_gemm_kernel<\(int\)192, \(int\)6>" -s 2 -c 1 -o $out/gemm_mlp1 \
    python tools/run_iteration.py --blocks 2 --eager > $out/ncu_mlp1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:tc_attn_kernel" -s 2 -c 1 -o $out/attn \
    python tools/run_iteration.py --blocks 2 --eager > $out/ncu_attn.log 2>&1
echo done

#!/bin/bash
# bench (both arms) + batched-scene mode + the sharded GPU tests
tag=${1:-r2b}
out=gpurun_out/$tag; mkdir -p $out
timeout 900 python bench.py --steps 10 --warmup 3 > $out/bench.json 2> $out/bench.err
timeout 600 python -m pytest tests/test_dist_gpu.py -q -x > $out/dist_gpu.log 2>&1; echo "rc=$?" >> $out/dist_gpu.log
timeout 900 python bench.py --scenes 8 --n 16 --steps 2 --warmup 1 > $out/bench_scenes.json 2> $out/bench_scenes.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $out/bench_ref.json 2> $out/bench_ref.err
lscpu > $out/lscpu.txt

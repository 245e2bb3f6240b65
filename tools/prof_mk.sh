#!/bin/bash
tag=${1:-pmk}
out=gpurun_out/$tag
mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:iter_kernel -s 0 -c 1 -o $out/mk python tools/run_iteration.py --blocks 4 --iters 1 --eager > $out/ncu.log 2>&1
echo done

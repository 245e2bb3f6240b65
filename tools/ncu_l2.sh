#!/bin/bash
# DRAM bytes / L2 hit rate of one persistent iteration (36 blocks) per ALPA_MK_FLAGS value
tag=${1:-l2}; shift
out=gpurun_out/$tag
mkdir -p $out
for f in "$@"; do
  ALPA_MK_FLAGS=$f timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
     --clock-control none -k regex:iter_kernel -s 0 -c 1 --csv python tools/run_iteration.py --blocks 36 --iters 1 --eager > $out/f$f.csv 2>&1
done
echo done

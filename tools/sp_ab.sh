#!/bin/bash
# Sweep-point A/B of env settings: tools/sp_ab.sh tag N K "ENV=.." "ENV=.." ...
tag=$1; n=$2; k=$3; shift 3
out=gpurun_out/$tag; mkdir -p $out
for setting in "$@"; do
  r=$(env $setting timeout 300 python tools/sweep_point.py $n $k 2>&1 | tail -1)
  echo "N=$n K=$k [$setting] $r" | tee -a $out/index.txt
done

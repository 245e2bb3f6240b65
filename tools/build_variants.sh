#!/bin/bash
# build A/B library variants into abl/<name>/ : tools/build_variants.sh name "-DX=1" [name "-DY=2" ...]
cd "$(dirname "$0")/../paper_2605_08975_b200"
while [ $# -gt 0 ]; do
  n=$1; f=$2; shift 2
  make -s -j8 BUILD=../abl/$n OUT=../abl/$n/libalpa_action.so EXTRA="$f" > /dev/null || exit 1
  echo "built abl/$n ($f): $(grep -A2 'iter_kernelILi192ELi128ELb0' ../abl/$n/mk.ptxas.log | grep spill)"
done

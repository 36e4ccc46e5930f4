#!/bin/bash
# ncu --set full of one kernel (regex $1) from a short bench run; report name $2.
# Usage: tools/gpu_ncu_kernel.sh <kernel-regex> <tag> [launch-skip] [bench args...]
K=$1; T=$2; S=${3:-1}; shift 3
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-scalar $@"
timeout 900 $CMD > gpurun_out/plain_$T.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_$T.log; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c 1 -f -o gpurun_out/prof_$T $CMD > gpurun_out/ncu_$T.log 2>&1
echo "ncu=$?"

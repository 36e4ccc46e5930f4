#!/bin/bash
# ncu --set full of the top kernels (one launch each), cfg2 bench command
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain_full.log 2>&1 || { echo "plain run failed"; exit 1; }
for K in reslice_k frame_scatter_k seal_k; do
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o gpurun_out/prof_$K $CMD > gpurun_out/ncu_$K.log 2>&1
  echo "$K=$?" >> gpurun_out/status.txt
done

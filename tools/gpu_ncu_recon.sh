#!/bin/bash
# ncu --set full on the reconstruct kernels (one launch each) of the cfg2 bench
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain_full.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"frame_scatter_k|seal_k" -s 0 -c 3 -o gpurun_out/prof_recon $CMD > gpurun_out/ncu_recon.log 2>&1; echo "ncu=$?"

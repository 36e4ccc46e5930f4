#!/bin/bash
# ncu --set full on the reconstruct kernels (one launch each) of the cfg2 bench
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-scalar"
timeout 900 $CMD > gpurun_out/plain_full.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-frame_count_k|frame_fill_k|seal_k}" -s ${NCU_S:-0} -c ${NCU_C:-3} -o gpurun_out/prof_${NCU_TAG:-recon} $CMD > gpurun_out/ncu_recon.log 2>&1; echo "ncu=$?"

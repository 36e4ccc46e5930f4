#!/bin/bash
# ncu --set full of the top reslice kernel and of the recon fill pass (cfg2 bench), one launch each
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-scalar"
timeout 900 $CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"reslice_fast_k" -s 1 -c 1 -o gpurun_out/prof_rs $CMD > gpurun_out/ncu_rs.log 2>&1; echo "ncu_rs=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"frame_run_k" -s 1 -c 1 -o gpurun_out/prof_fill $CMD > gpurun_out/ncu_fill.log 2>&1; echo "ncu_fill=$?"

#!/bin/bash
# ncu --set full of the cfg3 bucketed fill and placement kernels (one launch each)
mkdir -p gpurun_out
CMD="python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-scalar"
for spec in "frame_fill_k:0:fill" "bucket_place_k:0:place" "seal_k:0:seal" "frame_count_tab_k:0:count"; do
  K=${spec%%:*}; rest=${spec#*:}; SK=${rest%%:*}; T=${rest#*:}
  timeout 1200 ncu --set full --clock-control none -k regex:"$K" -s $SK -c 1 -f -o /tmp/c3_$T $CMD > gpurun_out/c3_ncu_$T.log 2>&1; echo "$T=$?"
  ncu -i /tmp/c3_$T.ncu-rep --page raw --csv > gpurun_out/c3_raw_$T.csv 2>/dev/null
done

#!/bin/bash
# Evidence capture: plain bench (cfg2), ncu launch list of our kernels, ncu --set full of the
# dominant kernels (one launch each).  Outputs in gpurun_out/ (summarised into profiles/).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "bench=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --exact --no-cpu-baseline --no-scalar > gpurun_out/bench_cfg2_exact.json 2> gpurun_out/bench_cfg2_exact.err; echo "bench_exact=$?" >> gpurun_out/status.txt
CMD="python bench.py --steps 5 --warmup 2 --no-cpu-baseline"
timeout 900 $CMD > gpurun_out/plain_cap.log 2>&1 || { echo "plain failed" >> gpurun_out/status.txt; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"reslice|prep_k|gate_k|pose_key_k|frame_count_k|frame_fill_k|seal_k|bin_cells|DeviceScan|DeviceReduce|compound|fill_|trilinear|merge|mufu|RadixSort|pack_coverage" \
  --csv --log-file gpurun_out/launches_cfg2.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launches=$?" >> gpurun_out/status.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"reslice_fast_k" -s 2 -c 1 \
  -o gpurun_out/full_reslice $CMD > gpurun_out/ncu_full_reslice.log 2>&1; echo "full_reslice=$?" >> gpurun_out/status.txt
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"frame_count_k|frame_fill_k|seal_k|compound_k" -s 4 -c 4 \
  -o gpurun_out/full_recon $CMD > gpurun_out/ncu_full_recon.log 2>&1; echo "full_recon=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt

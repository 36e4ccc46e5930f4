#!/bin/bash
# profiling pass: phase timings + ncu launch list of our kernels (cfg2)
mkdir -p gpurun_out
DARE_PROFILE=1 timeout 900 python bench.py --steps 10 --warmup 2 --no-cpu-baseline > gpurun_out/bench_prof.log 2> gpurun_out/bench_prof.err; echo "plain=$?" > gpurun_out/status.txt
timeout 900 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/plain_small.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"reslice_k|gate_k|scatter|seal_k|Scan|big_|compound|fill|trilinear" --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_run.log 2>&1; echo "ncu=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt

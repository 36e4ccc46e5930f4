#!/bin/bash
# large configs: cfg3 (8000 frames -> 512^3), cfg4 (trajectory reslices), reference arm cfg2.
# Plain runs (no DARE_PROFILE) for the JSON lines; a profiled cfg3 run for phase times.
mkdir -p gpurun_out
timeout 1500 python bench.py --config cfg3 --steps 10 --warmup 3 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "cfg3=$?" >> gpurun_out/status.txt
timeout 1500 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4=$?" >> gpurun_out/status.txt
DARE_PROFILE=1 timeout 1500 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-scalar > gpurun_out/bench_cfg3_prof.json 2> gpurun_out/bench_cfg3_prof.err; echo "cfg3_prof=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref_cfg2.json 2> gpurun_out/bench_ref_cfg2.err; echo "ref_cfg2=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt

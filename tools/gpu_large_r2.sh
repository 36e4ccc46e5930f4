#!/bin/bash
# cfg3 / cfg4 / cfg1 bench lines (recon phases on stderr with DARE_PROFILE)
mkdir -p gpurun_out
T=${1:-l}
DARE_PROFILE=1 timeout 1200 python bench.py --config cfg3 --steps 10 --warmup 3 --no-cpu-baseline --no-scalar > gpurun_out/bench_cfg3_$T.json 2> gpurun_out/bench_cfg3_$T.err; echo "cfg3=$?"
timeout 1200 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline --no-scalar > gpurun_out/bench_cfg4_$T.json 2> gpurun_out/bench_cfg4_$T.err; echo "cfg4=$?"
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 5 > gpurun_out/bench_cfg1_$T.json 2> gpurun_out/bench_cfg1_$T.err; echo "cfg1=$?"

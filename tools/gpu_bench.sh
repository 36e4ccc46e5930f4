#!/bin/bash
# GPU pass: parity tests + benches (args: extra bench args)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" > gpurun_out/status.txt
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 3 > gpurun_out/bench_cfg1.log 2>&1; echo "bench_cfg1=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --steps 30 --warmup 3 "$@" > gpurun_out/bench_cfg2.log 2>&1; echo "bench_cfg2=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt

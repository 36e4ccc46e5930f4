#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo "pytest=$rc" >> gpurun_out/status.txt
[ $rc -ne 0 ] && exit 1
DARE_PROFILE=1 timeout 1500 python bench.py --config cfg4 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt

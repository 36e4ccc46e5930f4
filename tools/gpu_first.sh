#!/bin/bash
# first GPU pass: tests, smoke, short benches
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" > gpurun_out/status.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 3 > gpurun_out/bench_cfg1.log 2>&1; echo "bench_cfg1=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --steps 30 --warmup 3 > gpurun_out/bench_cfg2.log 2>&1; echo "bench_cfg2=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt

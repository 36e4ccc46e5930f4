#!/bin/bash
# Round 2 pass: GPU tests (all, incl. the reference-scale hashes), smoke, the
# default bench line and the reference arm.  Usage: tools/gpu_r2.sh [tag]
T=${1:-a}
mkdir -p gpurun_out; rm -f gpurun_out/status_$T.txt
nvidia-smi --query-gpu=name,driver_version,memory.total --format=csv > gpurun_out/gpu_$T.txt 2>&1
lscpu > gpurun_out/lscpu_$T.txt 2>&1; free -g >> gpurun_out/lscpu_$T.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=15 > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest=$?" >> gpurun_out/status_$T.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke=$?" >> gpurun_out/status_$T.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench=$?" >> gpurun_out/status_$T.txt
timeout 900 python bench.py --impl reference --steps 10 --warmup 2 > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; echo "ref=$?" >> gpurun_out/status_$T.txt
cat gpurun_out/status_$T.txt

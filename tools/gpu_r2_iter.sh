#!/bin/bash
# Round 2 iteration: GPU tests (stop at first failure), then profiled bench
# lines (DARE_PROFILE phase events on stderr).  Usage: tools/gpu_r2_iter.sh tag [bench args]
T=${1:-it}; shift
mkdir -p gpurun_out; rm -f gpurun_out/status_$T.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -rf > gpurun_out/pytest_$T.log 2>&1; rc=$?; echo "pytest=$rc" >> gpurun_out/status_$T.txt
if [ $rc -ne 0 ]; then tail -40 gpurun_out/pytest_$T.log; cat gpurun_out/status_$T.txt; exit 1; fi
DARE_PROFILE=1 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench=$?" >> gpurun_out/status_$T.txt
DARE_PROFILE=1 DARE_NARROW_KEYS=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/bench_${T}_legacy.json 2> gpurun_out/bench_${T}_legacy.err; echo "legacy=$?" >> gpurun_out/status_$T.txt
cat gpurun_out/status_$T.txt

#!/bin/bash
# iteration pass: parity tests -> (only if green) profiled bench -> optional ncu full of reslice_k
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/bench_prof.log
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo "pytest=$rc" >> gpurun_out/status.txt
if [ $rc -ne 0 ]; then cat gpurun_out/status.txt; exit 1; fi
DARE_PROFILE=1 timeout 900 python bench.py --steps 20 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_prof.log 2> gpurun_out/bench_prof.err; rc=$?; echo "bench=$rc" >> gpurun_out/status.txt
if [ $rc -ne 0 ]; then cat gpurun_out/status.txt; exit 1; fi
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
if [ "$1" == "ncu" ]; then
timeout 900 $CMD > gpurun_out/plain_full.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-reslice_k}" -s 1 -c 1 -o gpurun_out/prof_${NCU_TAG:-reslice} $CMD > gpurun_out/ncu_${NCU_TAG:-reslice}.log 2>&1; echo "ncu=$?" >> gpurun_out/status.txt
fi
cat gpurun_out/status.txt

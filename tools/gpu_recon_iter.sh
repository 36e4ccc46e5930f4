#!/bin/bash
# Reconstruction iteration: parity (goldens, reference hashes, sampled cells at cfg2/cfg3), then
# DARE_PROFILE phase times of cfg2 and cfg3 builds.  Usage: tools/gpu_recon_iter.sh tag
T=${1:-rc}
mkdir -p gpurun_out; S=gpurun_out/status_$T.txt; rm -f $S
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_fullsize.py \
  tests/test_gpu_fullsize_cfg3.py -k "not reslice_patches and not trajectory" -x -q -p no:cacheprovider -rf \
  > gpurun_out/pytest_$T.log 2>&1; rc=$?; echo "pytest=$rc" >> $S
if [ $rc -ne 0 ]; then tail -30 gpurun_out/pytest_$T.log; cat $S; exit 1; fi
DARE_PROFILE=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-scalar > gpurun_out/bench_${T}_cfg2.json 2> gpurun_out/bench_${T}_cfg2.err; echo "cfg2=$?" >> $S
DARE_PROFILE=1 timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-scalar > gpurun_out/bench_${T}_cfg3.json 2> gpurun_out/bench_${T}_cfg3.err; echo "cfg3=$?" >> $S
cat $S
DARE_FILL_V1=1 DARE_PROFILE=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-scalar > gpurun_out/bench_${T}_cfg2_v1.json 2> gpurun_out/bench_${T}_cfg2_v1.err; echo "cfg2_v1=$?" >> $S
DARE_FILL_V1=1 DARE_PROFILE=1 timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-scalar > gpurun_out/bench_${T}_cfg3_v1.json 2> gpurun_out/bench_${T}_cfg3_v1.err; echo "cfg3_v1=$?" >> $S

#!/bin/bash
# Reconstruction iteration: parity (goldens, reference hashes, sampled cells at cfg2/cfg3), then
# DARE_PROFILE phase times of cfg2 and cfg3 builds, default and with an A/B switch.
# Usage: tools/gpu_recon_iter.sh tag [VAR=value]   (e.g. DARE_FILL_U8=0)
T=${1:-rc}; AB=${2:-DARE_NOTHING=1}
mkdir -p gpurun_out; S=gpurun_out/status_$T.txt; rm -f $S
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_fullsize.py \
  tests/test_gpu_fullsize_cfg3.py -k "not reslice_patches and not trajectory" -x -q -p no:cacheprovider -rf \
  > gpurun_out/pytest_$T.log 2>&1; rc=$?; echo "pytest=$rc" >> $S
if [ $rc -ne 0 ]; then tail -30 gpurun_out/pytest_$T.log; cat $S; exit 1; fi
for c in cfg2 cfg3; do
  DARE_PROFILE=1 timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-scalar > gpurun_out/bench_${T}_$c.json 2> gpurun_out/bench_${T}_$c.err; echo "$c=$?" >> $S
  env $AB DARE_PROFILE=1 timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-scalar > gpurun_out/bench_${T}_${c}_ab.json 2> gpurun_out/bench_${T}_${c}_ab.err; echo "${c}_ab=$?" >> $S
done
cat $S

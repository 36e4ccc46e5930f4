#!/bin/bash
# Direction-cluster index: parity (split tests, certified == exact, goldens,
# cfg3 / cfg4 slab-oracle patches) and cfg3 / cfg4 bench lines with and
# without it (DARE_ORIENT_SPLIT=0).  Usage: tools/gpu_split_iter.sh tag
T=${1:-sp}
mkdir -p gpurun_out; S=gpurun_out/status_$T.txt; rm -f $S
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_cfg3.py -x -q -p no:cacheprovider -rf \
  -k "direction_cluster or certified or acceptance or goldens or reslice_patches or trajectory or split or batch or concurrent" \
  > gpurun_out/pytest_$T.log 2>&1; rc=$?; echo "pytest=$rc" >> $S
if [ $rc -ne 0 ]; then tail -30 gpurun_out/pytest_$T.log; cat $S; exit 1; fi
for c in cfg3 cfg4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-scalar > gpurun_out/bench_${T}_$c.json 2> gpurun_out/bench_${T}_$c.err; echo "$c=$?" >> $S
  DARE_ORIENT_SPLIT=0 timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-scalar > gpurun_out/bench_${T}_${c}_nosplit.json 2> gpurun_out/bench_${T}_${c}_nosplit.err; echo "${c}_nosplit=$?" >> $S
done
cat $S

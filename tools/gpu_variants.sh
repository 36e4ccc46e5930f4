#!/bin/bash
# A/B of certified-kernel variants (DARE_FAST_VARIANT), plain bench runs, no profiler.
mkdir -p gpurun_out
for v in ${VARIANTS:-0 1 2 3 4}; do
  DARE_FAST_VARIANT=$v timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-scalar ${BENCH_ARGS} \
    > gpurun_out/var_$v.log 2> gpurun_out/var_$v.err
  echo "variant $v rc=$?"
done

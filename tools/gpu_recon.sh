#!/bin/bash
# parity tests, then profiled cfg2 + cfg3 bench runs (reconstruction phase times in *.err)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
DARE_PROFILE=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-scalar > gpurun_out/b2.json 2> gpurun_out/b2.err; echo "b2=$?"
DARE_PROFILE=1 timeout 1500 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-scalar > gpurun_out/b3.json 2> gpurun_out/b3.err; echo "b3=$?"

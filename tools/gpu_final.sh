#!/bin/bash
# Round-end evidence: tests, smoke, cfg2 capture (bench lines, launch list, ncu full of the
# top kernels), then cfg1 / cfg3 / cfg4 / reference-arm bench lines.
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/status.txt
bash tools/gpu_capture.sh > gpurun_out/capture.log 2>&1; echo "capture=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 3 > gpurun_out/bench_cfg1.json 2> gpurun_out/bench_cfg1.err; echo "cfg1=$?" >> gpurun_out/status.txt
bash tools/gpu_large.sh > gpurun_out/large.log 2>&1; echo "large=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt

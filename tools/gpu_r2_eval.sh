#!/bin/bash
# Evaluation harness + C client check on the GPU box: their GPU tests, the
# reference's own test files against the drop-in (incl. test_evaluation.py),
# and one cfg2 bench line with the evaluation leg.
mkdir -p gpurun_out; S=gpurun_out/ev2_status.txt; rm -f $S
timeout 900 python -m pytest tests/test_gpu_eval.py tests/test_c_abi_program.py -q -p no:cacheprovider -rf \
  > gpurun_out/ev2_pytest.log 2>&1; echo "pytest=$?" >> $S
bash tools/conformance.sh > gpurun_out/ev2_conformance.log 2>&1; echo "conformance=$?" >> $S
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/ev2_bench_cfg2.json 2> gpurun_out/ev2_bench_cfg2.err; echo "bench=$?" >> $S
cat $S

#!/bin/bash
# Last capture of the round: full GPU suite, smoke, conformance, bench lines.
mkdir -p gpurun_out; S=gpurun_out/f3_status.txt; rm -f $S
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=10 > gpurun_out/f3_pytest_gpu.log 2>&1; echo "pytest=$?" >> $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "smoke=$?" >> $S
bash tools/conformance.sh > gpurun_out/f3_conformance.log 2>&1; echo "conformance=$?" >> $S
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f3_bench_cfg2.json 2> gpurun_out/f3_bench_cfg2.err; echo "bench=$?" >> $S
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/f3_bench_ref_cfg2.json 2> gpurun_out/f3_bench_ref_cfg2.err; echo "ref=$?" >> $S
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 5 > gpurun_out/f3_bench_cfg1.json 2> gpurun_out/f3_bench_cfg1.err; echo "cfg1=$?" >> $S
timeout 1500 python bench.py --config cfg3 --steps 10 --warmup 3 > gpurun_out/f3_bench_cfg3.json 2> gpurun_out/f3_bench_cfg3.err; echo "cfg3=$?" >> $S
timeout 1500 python bench.py --config cfg4 --steps 10 --warmup 3 --no-scalar > gpurun_out/f3_bench_cfg4.json 2> gpurun_out/f3_bench_cfg4.err; echo "cfg4=$?" >> $S
cat $S

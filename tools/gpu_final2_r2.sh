#!/bin/bash
# Post-index capture: full GPU suite, smoke, bench lines (cfg2 default, reference
# arm, cfg1, cfg3, cfg4), ncu --set full of the cfg3 index kernel.
mkdir -p gpurun_out; S=gpurun_out/f2_status.txt; rm -f $S
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=10 > gpurun_out/f2_pytest_gpu.log 2>&1; echo "pytest=$?" >> $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; echo "smoke=$?" >> $S
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f2_bench_cfg2.json 2> gpurun_out/f2_bench_cfg2.err; echo "bench=$?" >> $S
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/f2_bench_ref_cfg2.json 2> gpurun_out/f2_bench_ref_cfg2.err; echo "ref=$?" >> $S
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 5 > gpurun_out/f2_bench_cfg1.json 2> gpurun_out/f2_bench_cfg1.err; echo "cfg1=$?" >> $S
timeout 1500 python bench.py --config cfg3 --steps 10 --warmup 3 > gpurun_out/f2_bench_cfg3.json 2> gpurun_out/f2_bench_cfg3.err; echo "cfg3=$?" >> $S
timeout 1500 python bench.py --config cfg4 --steps 10 --warmup 3 --no-scalar > gpurun_out/f2_bench_cfg4.json 2> gpurun_out/f2_bench_cfg4.err; echo "cfg4=$?" >> $S
CMD="python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline --no-scalar"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"reslice_fast_k" -s 4 -c 1 -f -o /tmp/f2_split $CMD > gpurun_out/f2_ncu_split.log 2>&1; echo "ncu_split=$?" >> $S
ncu -i /tmp/f2_split.ncu-rep --page raw --csv > gpurun_out/f2_raw_split.csv 2>/dev/null
ncu -i /tmp/f2_split.ncu-rep --page details --csv > gpurun_out/f2_details_split.csv 2>/dev/null
cat $S

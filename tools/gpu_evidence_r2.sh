#!/bin/bash
# Round-2 evidence capture: GPU tests, smoke, bench lines (cfg2 default, reference
# arm, cfg1/cfg3/cfg4), ncu launch list of the cfg2 bench, ncu --set full of the
# dominant kernels (one launch each).  Everything lands in gpurun_out/ev_*.
mkdir -p gpurun_out; S=gpurun_out/ev_status.txt; rm -f $S
nvidia-smi > gpurun_out/ev_nvidia_smi.txt 2>&1; lscpu > gpurun_out/ev_lscpu.txt 2>&1
if [ "$1" != "nobench" ]; then
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=20 > gpurun_out/ev_pytest_gpu.log 2>&1; echo "pytest=$?" >> $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "smoke=$?" >> $S
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/ev_bench_cfg2.json 2> gpurun_out/ev_bench_cfg2.err; echo "bench=$?" >> $S
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ev_bench_ref_cfg2.json 2> gpurun_out/ev_bench_ref_cfg2.err; echo "ref=$?" >> $S
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 5 > gpurun_out/ev_bench_cfg1.json 2> gpurun_out/ev_bench_cfg1.err; echo "cfg1=$?" >> $S
timeout 1500 python bench.py --config cfg3 --steps 10 --warmup 3 > gpurun_out/ev_bench_cfg3.json 2> gpurun_out/ev_bench_cfg3.err; echo "cfg3=$?" >> $S
timeout 1500 python bench.py --config cfg4 --steps 10 --warmup 3 --no-scalar > gpurun_out/ev_bench_cfg4.json 2> gpurun_out/ev_bench_cfg4.err; echo "cfg4=$?" >> $S
fi
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches_cfg2.csv $CMD > gpurun_out/ev_ncu_launches.log 2>&1; echo "launches=$?" >> $S
for spec in "reslice_fast_k:4:reslice" "frame_count_tab_k:1:count" "frame_fill_k:1:fill" "seal_k:1:seal" "compound2_k:1:compound" "fill_pass_k:0:fillpass" "trilinear_k:0:trilinear" "reslice_fallback_k:4:fallback" "prep_k:4:prep"; do
  K=${spec%%:*}; rest=${spec#*:}; SK=${rest%%:*}; T=${rest#*:}
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $SK -c 1 -f -o /tmp/ev_prof_$T $CMD > gpurun_out/ev_ncu_$T.log 2>&1; echo "ncu_$T=$?" >> $S
  # exports only (gpurun copies back <= 64 MiB): raw metrics, details, SASS source page of the hot kernels
  ncu -i /tmp/ev_prof_$T.ncu-rep --page raw --csv > gpurun_out/ev_raw_$T.csv 2>/dev/null
  ncu -i /tmp/ev_prof_$T.ncu-rep --page details --csv > gpurun_out/ev_details_$T.csv 2>/dev/null
  case $T in reslice|seal|count|fill|compound) ncu -i /tmp/ev_prof_$T.ncu-rep --page source --csv --print-source sass > gpurun_out/ev_sass_$T.csv 2>/dev/null;; esac
done
du -sh gpurun_out
cat $S

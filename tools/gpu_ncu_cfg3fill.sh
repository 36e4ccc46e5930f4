bash tools/gpu_ncu_kernel.sh frame_fill_k cfg3fill 3 --config cfg3
ncu -i gpurun_out/prof_cfg3fill.ncu-rep --page details --csv > gpurun_out/cfg3fill_details.csv 2>/dev/null
ncu -i gpurun_out/prof_cfg3fill.ncu-rep --page raw --csv > gpurun_out/cfg3fill_raw.csv 2>/dev/null
ncu -i gpurun_out/prof_cfg3fill.ncu-rep --page source --csv --print-source sass > gpurun_out/cfg3fill_sass.csv 2>/dev/null
ls -la gpurun_out/prof_cfg3fill.ncu-rep; tail -3 gpurun_out/ncu_cfg3fill.log

# source-level ncu capture of ONE C5 mode-1 fused power step (second launch of one_power_step.py)
ncu --set full --import-source on --clock-control none -k regex:fused_power_kernel -s 1 -c 1 \
    -o gpurun_out/fused_c5s python scripts/one_power_step.py 1000 1000000 60 2 > gpurun_out/ncu_fused_c5s.log 2>&1
ncu -i gpurun_out/fused_c5s.ncu-rep --page source --csv --print-source sass > gpurun_out/fused_src_c5.csv 2>/dev/null
ncu -i gpurun_out/fused_c5s.ncu-rep --page raw --csv > gpurun_out/fused_raw_c5.csv 2>/dev/null
tail -1 gpurun_out/ncu_fused_c5s.log

ncu --set full --import-source on --clock-control none -k regex:fused_power_kernel -s 15 -c 1 \
    -o gpurun_out/fused_c5s python scripts/prof_solve.py c5 1 > gpurun_out/ncu_fused_c5s.log 2>&1
ncu -i gpurun_out/fused_c5s.ncu-rep --page source --csv --print-source sass > gpurun_out/fused_src_c5.csv 2>/dev/null
tail -1 gpurun_out/ncu_fused_c5s.log

# full ncu capture of one C5 mode-1 fused power step (launch index 1 of the timed solve)
ncu --set full --import-source on --clock-control none -k regex:fused_power_kernel -s 15 -c 1 \
    -o gpurun_out/fused_c5 python scripts/prof_solve.py c5 1 > gpurun_out/ncu_fused_c5.log 2>&1
ncu -i gpurun_out/fused_c5.ncu-rep --page details --csv > gpurun_out/fused_details_c5.csv 2>/dev/null
ncu -i gpurun_out/fused_c5.ncu-rep --page raw --csv > gpurun_out/fused_raw_c5.csv 2>/dev/null
tail -2 gpurun_out/ncu_fused_c5.log

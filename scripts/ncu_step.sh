# ncu --set full of one cluster small-solve launch (C5, 9th step_kernel launch of the timed solve),
# densest warp-state sampling (every 32 cycles)
ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:step_kernel -s 8 -c 1 \
    -o gpurun_out/step_kernel python scripts/prof_solve.py c5 1 > gpurun_out/ncu_step.log 2>&1
ncu -i gpurun_out/step_kernel.ncu-rep --page source --csv --print-source sass > gpurun_out/step_src.csv 2>/dev/null
ncu -i gpurun_out/step_kernel.ncu-rep --page raw --csv > gpurun_out/step_raw.csv 2>/dev/null
tail -3 gpurun_out/ncu_step.log

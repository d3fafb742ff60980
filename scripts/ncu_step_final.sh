ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 5 -c 1 -o gpurun_out/step_final python scripts/one_solve.py c5 > gpurun_out/ncu_step_final.log 2>&1
ncu -i gpurun_out/step_final.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/step_final_src.csv 2>/dev/null
ncu -i gpurun_out/step_final.ncu-rep --page raw --csv > gpurun_out/step_final_raw.csv 2>/dev/null
tail -2 gpurun_out/ncu_step_final.log

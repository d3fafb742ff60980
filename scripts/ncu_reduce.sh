ncu --set full --import-source on --clock-control none --cache-control none -k regex:reduce_gram -s 2 -c 1 -o gpurun_out/reduce_c5 python scripts/one_solve.py c5 > /dev/null 2>&1
ncu -i gpurun_out/reduce_c5.ncu-rep --page raw --csv > gpurun_out/reduce_raw.csv 2>/dev/null
ncu -i gpurun_out/reduce_c5.ncu-rep --page source --csv --print-source sass > gpurun_out/reduce_src.csv 2>/dev/null
ncu -i gpurun_out/reduce_c5.ncu-rep --page details --csv > gpurun_out/reduce_details.csv 2>/dev/null
echo done

# ncu --set full of ONE C5 mode-1 shaped power step on the pair engine (second launch of one_power_step.py)
ncu --set full --import-source on --clock-control none -k regex:pair_power_kernel -s 1 -c 1 \
    -o gpurun_out/pair_c5 python scripts/one_power_step.py 1000 1000000 60 2 > gpurun_out/ncu_pair_c5.log 2>&1
ncu -i gpurun_out/pair_c5.ncu-rep --page source --csv --print-source sass > gpurun_out/pair_src_c5.csv 2>/dev/null
ncu -i gpurun_out/pair_c5.ncu-rep --page raw --csv > gpurun_out/pair_raw_c5.csv 2>/dev/null
ncu -i gpurun_out/pair_c5.ncu-rep --page details --csv > gpurun_out/pair_details_c5.csv 2>/dev/null
tail -2 gpurun_out/ncu_pair_c5.log
python scripts/ncu_summary.py gpurun_out/pair_raw_c5.csv

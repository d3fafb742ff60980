# ncu --set full of one fused power-step launch (config $1, launch index $2)
cfg=${1:-c4}; idx=${2:-3}
ncu --set full --import-source on --clock-control none -k regex:fused_power_kernel -s $idx -c 1 \
    -o gpurun_out/fused_$cfg python scripts/prof_solve.py $cfg 1 > gpurun_out/ncu_fused_$cfg.log 2>&1
ncu -i gpurun_out/fused_$cfg.ncu-rep --page source --csv --print-source sass > gpurun_out/fused_src_$cfg.csv 2>/dev/null
ncu -i gpurun_out/fused_$cfg.ncu-rep --page details --csv > gpurun_out/fused_details_$cfg.csv 2>/dev/null
tail -2 gpurun_out/ncu_fused_$cfg.log

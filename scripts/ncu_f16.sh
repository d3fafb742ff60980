# ncu of the fp16 pair power step (C5 mode 1, first power step of one C5 solve) + a lag sweep
ncu --set full --import-source on --clock-control none -k regex:pair_power_kernel -s 1 -c 1 \
    -o gpurun_out/pair16_c5 python scripts/one_solve.py c5 > gpurun_out/ncu_pair16_c5.log 2>&1
ncu -i gpurun_out/pair16_c5.ncu-rep --page source --csv --print-source sass > gpurun_out/pair16_src_c5.csv 2>/dev/null
ncu -i gpurun_out/pair16_c5.ncu-rep --page raw --csv > gpurun_out/pair16_raw_c5.csv 2>/dev/null
tail -2 gpurun_out/ncu_pair16_c5.log
python scripts/ncu_summary.py gpurun_out/pair16_raw_c5.csv
for lag in 0 1 2 3 4; do
  echo "== lag $lag"
  RTK_PAIR_LAG=$lag ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active \
     --clock-control none -k regex:pair_power_kernel -s 1 -c 2 --csv python scripts/one_solve.py c5 2>/dev/null | grep -v "^==" | tail -6
done

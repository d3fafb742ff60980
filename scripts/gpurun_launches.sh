# ncu launch list (per-kernel device time) of one profiled solve: python scripts/prof_solve.py <cfg> 1
cfg=${1:-c5}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv \
    python scripts/prof_solve.py $cfg 1 > gpurun_out/ncu_launch_$cfg.log 2>&1
python scripts/launch_summary.py gpurun_out/launches_$cfg.csv > gpurun_out/launch_summary_$cfg.txt
cat gpurun_out/launch_summary_$cfg.txt

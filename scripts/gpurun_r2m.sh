# round-2 closing evidence with graph replay: GPU suite, smoke, bench, launch list, ncu of the power step,
# per-launch pair-engine times of one C5 solve, config table
set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2m.json 2> gpurun_out/bench_r2m.err; echo bench rc $?
cat gpurun_out/bench_r2m.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r2m.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_bench_r2m.log 2>&1; echo ncu rc $?
python scripts/launch_summary.py gpurun_out/launches_r2m.csv > gpurun_out/launch_summary_r2m.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pair_power_kernel -s 1 -c 1 \
    -o gpurun_out/pair16_r2m python scripts/one_solve.py c5 > gpurun_out/ncu_pair16_r2m.log 2>&1; echo ncu full rc $?
ncu -i gpurun_out/pair16_r2m.ncu-rep --page raw --csv > gpurun_out/pair16_raw_r2m.csv 2>/dev/null
python scripts/ncu_summary.py gpurun_out/pair16_raw_r2m.csv > gpurun_out/ncu_pair16_summary_r2m.txt
rm -f gpurun_out/pair16_raw_r2m.csv
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:pair_power_kernel --csv --log-file gpurun_out/pair_modes_r2m.csv python scripts/one_solve.py c5 > /dev/null 2>&1
python scripts/ncu_pair_modes.py gpurun_out/pair_modes_r2m.csv > gpurun_out/pair_modes_r2m.md
timeout 900 python scripts/config_table.py > gpurun_out/configs_r2m.md 2> gpurun_out/configs_r2m.err; cat gpurun_out/configs_r2m.md

# round-2 final evidence: GPU suite, smoke, bench line, launch list, pair-engine launches of one C5
# solve, config table, step clocks
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err; echo bench rc $?
cat gpurun_out/bench_r2c.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r2c.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_bench_r2c.log 2>&1; echo ncu rc $?
python scripts/launch_summary.py gpurun_out/launches_r2c.csv > gpurun_out/launch_summary_r2c.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:pair_power_kernel --csv --log-file gpurun_out/pair_modes_r2c.csv python scripts/one_solve.py c5 > gpurun_out/ncu_pair_modes_r2c.log 2>&1
python scripts/ncu_pair_modes.py gpurun_out/pair_modes_r2c.csv > gpurun_out/pair_modes_r2c.md
timeout 900 python scripts/config_table.py > gpurun_out/configs_r2c.md 2> gpurun_out/configs_r2c.err; cat gpurun_out/configs_r2c.md
for c in c5 c3 c4; do echo "== $c"; timeout 120 python scripts/step_clocks.py $c; done > gpurun_out/step_clocks_r2c.txt 2>&1

# round-2 (second half) evidence: bench line, launch list, pair-engine launches of one C5 solve
# (sketch / power / shrink: time + DRAM bytes), the five-config table, step-kernel phase clocks
set -x
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo bench rc $?
cat gpurun_out/bench_r2b.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r2b.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_bench_r2b.log 2>&1; echo ncu rc $?
python scripts/launch_summary.py gpurun_out/launches_r2b.csv > gpurun_out/launch_summary_r2b.txt 2>&1
head -30 gpurun_out/launch_summary_r2b.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:pair_power_kernel --csv --log-file gpurun_out/pair_modes_r2b.csv python scripts/one_solve.py c5 > gpurun_out/ncu_pair_modes.log 2>&1
python scripts/ncu_pair_modes.py gpurun_out/pair_modes_r2b.csv | tee gpurun_out/pair_modes_r2b.md
timeout 900 python scripts/config_table.py > gpurun_out/configs_r2b.md 2> gpurun_out/configs_r2b.err; cat gpurun_out/configs_r2b.md
for c in c5 c3 c4; do echo "== $c"; timeout 120 python scripts/step_clocks.py $c; done > gpurun_out/step_clocks_r2b.txt 2>&1

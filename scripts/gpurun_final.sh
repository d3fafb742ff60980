# round-2 evidence: bench line, launch list of the bench command, ncu --set full of the pair engine
# (one C5 mode-1 power step), the five-config table
set -x
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc $?
cat gpurun_out/bench_final.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_bench_final.log 2>&1; echo ncu rc $?
python scripts/launch_summary.py gpurun_out/launches_final.csv > gpurun_out/launch_summary_final.txt 2>&1
head -30 gpurun_out/launch_summary_final.txt
timeout 600 bash scripts/ncu_pair.sh
timeout 900 python scripts/config_table.py > gpurun_out/configs_final.md 2> gpurun_out/configs_final.err; cat gpurun_out/configs_final.md

# round-end style validation: GPU tests, bench line, ncu launch list of the bench command,
# and one ncu --set full capture of the C5 mode-1 fused power step
set -x
timeout 700 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
cat gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_bench.log 2>&1; echo ncu rc $?
python scripts/launch_summary.py gpurun_out/launches_bench.csv > gpurun_out/launch_summary_bench.txt 2>&1
head -25 gpurun_out/launch_summary_bench.txt
timeout 600 bash scripts/ncu_fused_src.sh; echo ncu full rc $?

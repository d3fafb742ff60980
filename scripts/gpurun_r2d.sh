# round-2 re-entry check: GPU suite, bench line, config table, step clocks
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2d.json 2> gpurun_out/bench_r2d.err; echo bench rc $?
cat gpurun_out/bench_r2d.json
timeout 900 python scripts/config_table.py > gpurun_out/configs_r2d.md 2> gpurun_out/configs_r2d.err; cat gpurun_out/configs_r2d.md
for c in c5 c3 c4; do echo "== $c"; timeout 120 python scripts/step_clocks.py $c; done > gpurun_out/step_clocks_r2d.txt 2>&1

# round 2, first call: box facts, full GPU test suite (parity incl. full-size C5), bench line
set -x
free -g; nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rf -s > gpurun_out/pytest_gpu_r2a.log 2>&1; echo pytest rc $?
grep -E "passed|failed|elementwise|C5|FAIL|Error" gpurun_out/pytest_gpu_r2a.log | tail -60
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo bench rc $?
cat gpurun_out/bench_r2a.json; tail -5 gpurun_out/bench_r2a.err

set -x
timeout 1500 python -m pytest tests -m gpu -q -rf -s > gpurun_out/pytest_gpu_r2b.log 2>&1; echo pytest rc $?
grep -E "passed|failed|C5 full|FAIL|Error" gpurun_out/pytest_gpu_r2b.log | tail -20
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err; echo bench rc $?
cat gpurun_out/bench_r2b.json; tail -3 gpurun_out/bench_r2b.err

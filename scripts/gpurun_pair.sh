timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "fused" 2>&1 | tail -1
for i in 1 2 3; do timeout 60 python scripts/one_power_step.py 1000 1000000 60 20 | tail -1; done

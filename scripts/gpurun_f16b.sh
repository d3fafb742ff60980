set -x
timeout 300 python scripts/f16_probe2.py
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "f16 or power_step" 2>&1 | tail -4
for f in 0 1; do RTK_POWER_F16=$f timeout 120 python scripts/one_power_step.py 1000 1000000 60 10 2>&1 | tail -1; done
for f in 1 0; do RTK_PAIR_F16=$f timeout 300 python scripts/prof_solve.py c5 2>&1 | tail -1; done
for f in 1 0; do RTK_PAIR_F16=$f timeout 300 python scripts/prof_solve.py c3 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4

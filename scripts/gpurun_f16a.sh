# fp16 pair engine: kernel tests, timing A/B of the C5 mode-1 power step, a solve parity subset
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "f16" 2>&1 | tail -15
for f in 0 1; do RTK_POWER_F16=$f timeout 120 python scripts/one_power_step.py 1000 1000000 60 10; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c5_launch or fused_sketch" 2>&1 | tail -5
for f in 1 0; do RTK_PAIR_F16=$f timeout 300 python scripts/prof_solve.py c5 2>&1 | tail -8; done

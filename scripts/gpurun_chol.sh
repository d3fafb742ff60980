# blocked 8x8 Cholesky + inverse in the step kernel: parity, phase clocks, A/B
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for c in c5 c4; do RTK_CHOL=1 timeout 120 python scripts/step_clocks.py $c 2>&1 | grep "step [15]:" | head -4; done
for ch in 1 0; do for c in c5 c3 c4; do RTK_CHOL=$ch timeout 300 python scripts/prof_solve.py $c 3 2>&1 | tail -1; done; done

# RTK-GAUSS-2 (binary32 Box-Muller): bit-exactness vs the oracle, full GPU suite, timings
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "omega or sketch" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c5 c3 c4 c1; do timeout 300 python scripts/prof_solve.py $c 5 2>&1 | tail -1 | cut -c1-220; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:omega_planes -c 3 --csv python scripts/one_solve.py c5 2>/dev/null | grep -v "^==" | grep -o '"[0-9.]*"$'

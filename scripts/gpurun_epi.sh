timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "f16" 2>&1 | tail -2
for r in 1 2; do echo -n "power: "; ncu --metrics gpu__time_duration.sum --clock-control none -k regex:pair_power_kernel -s 1 -c 3 --csv python scripts/one_solve.py c5 2>/dev/null | grep -v "^==" | grep -o '"[0-9.]*"$' | tr '\n' ' '; echo; done
timeout 300 python scripts/prof_solve.py c5 5 2>&1 | tail -1 | cut -c1-150

set -x
for lag in 0 2 4; do RTK_PAIR_LAG=$lag timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:pair_power_kernel -s 1 -c 2 --csv python scripts/one_solve.py c5 2>/dev/null | grep -v "^==" | awk -F'","' '{print $(NF-2), $NF}' | tail -4; done
timeout 300 python scripts/prof_solve.py c5 3 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "f16" 2>&1 | tail -2

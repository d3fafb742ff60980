timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r2c.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/pytest_gpu_r2c.log
timeout 120 python scripts/prof_solve.py c5 3
timeout 120 python scripts/prof_solve.py c3 3
RTK_PAIR=1 timeout 120 python scripts/prof_solve.py c3 3

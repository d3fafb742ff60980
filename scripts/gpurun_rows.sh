for r in 1 2; do for rows in 64 32 48; do echo -n "rows=$rows "; RTK_STEP_ROWS=$rows timeout 300 python scripts/prof_solve.py c5 5 2>&1 | tail -1 | cut -c1-60,150-260; done; done
RTK_STEP_ROWS=32 timeout 120 python scripts/step_clocks.py c5 2>&1 | grep "step [15]:" | head -2
RTK_STEP_ROWS=32 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c5 or f16 or garbage" 2>&1 | tail -2

RTK_CHOL=2 timeout 120 python scripts/one_solve.py c5 2>&1 | grep "chol_inv prof" | grep -v "init 0 " | sed -n '1p;3p;14p'
for ch in 0 1; do for c in c5 c3; do echo -n "chol=$ch "; RTK_CHOL=$ch timeout 300 python scripts/prof_solve.py $c 5 2>&1 | tail -1 | cut -c1-60,170-260; done; done
for ch in 0 1; do echo "chol=$ch"; RTK_CHOL=$ch timeout 120 python scripts/step_clocks.py c5 2>&1 | grep "step 1:" | head -3; done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2

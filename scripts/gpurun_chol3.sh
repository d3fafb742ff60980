bash scripts/gpurun_chol2.sh 2>&1 | grep -v "init 0 " | tail -3
for rep in 1 2; do for ch in 0 1; do for c in c5 c3 c4; do echo -n "chol=$ch "; RTK_CHOL=$ch timeout 300 python scripts/prof_solve.py $c 5 2>&1 | tail -1; done; done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2

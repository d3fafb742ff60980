for r in 1 2; do for g in 1 0; do for c in c5 c3 c4; do echo -n "gbar=$g "; RTK_STEP_GBAR=$g timeout 300 python scripts/prof_solve.py $c 5 2>&1 | tail -1 | cut -c1-60,160-260; done; done; done
bash scripts/gpurun_reduce.sh | grep step | head -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2

timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash scripts/gpurun_reduce.sh | grep reduce | head -4 | cut -c1-20,120-200
for r in 1 2; do for c in c5 c3; do timeout 300 python scripts/prof_solve.py $c 5 2>&1 | tail -1 | cut -c1-60,150-260; done; done

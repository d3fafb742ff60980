set -x
bash scripts/gpurun_reduce.sh | head -8
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c5 c3 c4; do timeout 300 python scripts/prof_solve.py $c 5 2>&1 | tail -1 | cut -c1-220; done

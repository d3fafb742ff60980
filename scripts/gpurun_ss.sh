timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config_parity or random_shapes or edge or bitwise or exact" 2>&1 | tail -3
for c in c1 c2; do timeout 120 python scripts/prof_solve.py $c 5; RTK_FUSED_STRIDED=0 timeout 120 python scripts/prof_solve.py $c 5; done

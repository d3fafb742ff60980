# pair-engine shrink: new test, parity suite, C5 shrink timing A/B
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pair_shrink" 2>&1 | tail -3
for e in 0 1; do echo "RTK_PAIR_SHRINK=$e"; RTK_PAIR_SHRINK=$e timeout 120 python scripts/prof_solve.py c5 3 2>&1 | tail -1; RTK_PAIR_SHRINK=$e timeout 120 python scripts/prof_solve.py c3 3 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2

RTK_CHOL=2 timeout 120 python scripts/one_solve.py c5 2>&1 | grep "chol_inv prof" | head -40

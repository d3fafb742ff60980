# pair-engine sketch: focused tests, C5/C3 sketch timing A/B, then the full GPU suite
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_sketch or c5_launch" 2>&1 | tail -3
for e in 0 1; do echo "RTK_PAIR_SKETCH=$e"; RTK_PAIR_SKETCH=$e timeout 120 python scripts/prof_solve.py c5 3 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2

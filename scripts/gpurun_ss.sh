timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "config_parity and fused" 2>&1 | tail -1
timeout 120 python scripts/step_clocks.py c5 | grep -E "mode 1"
for c in c5 c4 c3; do timeout 120 python scripts/prof_solve.py $c 3; done

for c in c5 c3 c4; do echo "== $c"; timeout 120 python scripts/step_clocks.py $c; done
timeout 120 python scripts/prof_solve.py c3 3 2>&1 | tail -12
timeout 120 python scripts/prof_solve.py c4 3 2>&1 | tail -12

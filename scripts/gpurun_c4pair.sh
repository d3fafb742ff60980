for pr in "" 1; do for c in c4 c3 c1 c2; do echo -n "RTK_PAIR=$pr "; RTK_PAIR=$pr timeout 300 python scripts/prof_solve.py $c 5 2>&1 | tail -1 | cut -c1-230; done; done

# small-solver changes: phase clocks (new vs RTK_TRI_INV=block), GPU tests, C5 bench
for c in c5 c4; do echo "== $c"; timeout 120 python scripts/step_clocks.py $c | sed -n '1,2p;6,7p'; echo "-- block"; RTK_TRI_INV=block timeout 120 python scripts/step_clocks.py $c | sed -n '1,2p;6,7p'; done
for c in c3 c4 c5; do timeout 120 python scripts/prof_solve.py $c 3 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], d.get('breakdown_ms_per_step'))"

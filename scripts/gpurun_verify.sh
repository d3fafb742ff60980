# full GPU test suite + phase clocks + C5 bench + config timings (one call)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 120 python scripts/step_clocks.py c5 | sed -n "1,2p;6p;12p;18p"
timeout 120 python scripts/step_clocks.py c3 | sed -n "4p"
for c in c3 c4 c5; do timeout 120 python scripts/prof_solve.py $c 3 2>&1 | tail -1; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['ms_per_step'], d.get('breakdown_ms_per_step'), d['clocks'])"

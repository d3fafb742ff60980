# early PDL trigger (RTK_PDL_TRIGGER): A/B device time of the public-API solve, then the GPU suite
for r in 1 2; do for c in c5 c4 c3 c1; do for t in 0 1; do
  echo "$c trigger=$t $(RTK_PDL_TRIGGER=$t timeout 200 python scripts/graph_ab.py $c 10 1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["direct"])')"
done; done; done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2

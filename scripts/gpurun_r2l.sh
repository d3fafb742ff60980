# A/B: graph replay on C5 (RTK_GRAPH=0 vs default), PDL inside graphs, early reduce_gram trigger
set -x
timeout 600 python scripts/env_ab.py RTK_GRAPH 0 c5 20 6
timeout 600 python scripts/env_ab.py RTK_PDL 0 c5 20 3
RTK_GRAPH=0 timeout 600 python scripts/env_ab.py RTK_PDL 0 c5 20 3
for c in c4 c3 c5; do timeout 600 python scripts/env_ab.py RTK_RG_EARLY 1 $c 20 4; done
timeout 300 python -m pytest tests/test_gpu_graph.py -q -x 2>&1 | tail -2
RTK_RG_EARLY=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2

# graph replay: new tests, the whole GPU suite, A/B timing per config
set -x
timeout 600 python -m pytest tests/test_gpu_graph.py -x -q 2>&1 | tail -15
for c in c1 c2 c3 c4 c5; do timeout 300 python scripts/graph_ab2.py $c 20 3; done 2>&1 | tee gpurun_out/graph_ab2_r2i.txt
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5

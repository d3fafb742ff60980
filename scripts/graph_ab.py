"""A/B: direct enqueue vs CUDA-graph replay of the public-API solve, alternating blocks of reps.
python scripts/graph_ab.py [c5] [reps] [rounds]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2506_04840_b200 as rt  # noqa: E402
from workloads import CONFIGS, make_config_tensor_torch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
c = CONFIGS[name]
A = make_config_tensor_torch(name)
fn = rt.rsthosvd if c["algo"] == "rsthosvd" else rt.rthosvd
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    out = fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"])
    for _ in range(3):
        fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"], out=out)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"], out=out)
torch.cuda.synchronize()


def timed(f):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


res = {"config": name, "direct": [], "graph": []}
for _ in range(rounds):
    res["direct"].append(round(timed(lambda: fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"], out=out)), 4))
    res["graph"].append(round(timed(g.replay), 4))
print(json.dumps(res))

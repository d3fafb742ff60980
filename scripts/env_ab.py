"""A/B of an RTK_* switch: back-to-back device ms per solve with VAR unset vs VAR=VAL, alternating blocks,
public API with reused outputs (graph replay on; the switch is part of the graph key).
python scripts/env_ab.py RTK_RG_EARLY 1 c4 [reps] [rounds]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2506_04840_b200 as rt  # noqa: E402
from workloads import CONFIGS, make_config_tensor_torch  # noqa: E402

var, val = sys.argv[1], sys.argv[2]
name = sys.argv[3] if len(sys.argv) > 3 else "c4"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 3
c = CONFIGS[name]
A = make_config_tensor_torch(name)
seq = c["algo"] == "rsthosvd"
out = rt.solve(A, c["ranks"], c["p"], c["q"], c["omega_seed"], sequential=seq)


def timed(on):
    if on:
        os.environ[var] = val
    else:
        os.environ.pop(var, None)
    for _ in range(3):
        rt.solve(A, c["ranks"], c["p"], c["q"], c["omega_seed"], sequential=seq, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        rt.solve(A, c["ranks"], c["p"], c["q"], c["omega_seed"], sequential=seq, out=out)
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)


res = {"config": name, "var": f"{var}={val}", "off": [], "on": []}
for _ in range(rounds):
    res["off"].append(timed(False))
    res["on"].append(timed(True))
print(json.dumps(res))

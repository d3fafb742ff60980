"""A/B: solve time with the shift (Alg. 4) vs alpha = 0 (Alg. 2), alternating blocks, to see how much
of the deferred shift update (alpha_kernel on the side stream) sits on the critical path.
python scripts/probe_shift_ab.py c4 [reps] [rounds]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2506_04840_b200 as rt  # noqa: E402
from workloads import CONFIGS, make_config_tensor_torch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 3
c = CONFIGS[name]
A = make_config_tensor_torch(name)
seq = c["algo"] == "rsthosvd"
out = rt.solve(A, c["ranks"], c["p"], c["q"], c["omega_seed"], sequential=seq)
torch.cuda.synchronize()


def timed(shift):
    for _ in range(2):
        rt.solve(A, c["ranks"], c["p"], c["q"], c["omega_seed"], sequential=seq, shift=shift, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        rt.solve(A, c["ranks"], c["p"], c["q"], c["omega_seed"], sequential=seq, shift=shift, out=out)
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)


res = {"config": name, "shift": [], "noshift": []}
for _ in range(rounds):
    res["shift"].append(timed(True))
    res["noshift"].append(timed(False))
print(json.dumps(res))

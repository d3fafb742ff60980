"""Capture one rtk solve in a CUDA graph (torch.cuda.CUDAGraph) and replay it: checks that the
library's launch sequence is capturable (no host sync inside a solve) and times replay vs eager.

python scripts/graph_capture.py [c1]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_04840_b200 as rt  # noqa: E402
from workloads import CONFIGS, make_config_tensor  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
c = CONFIGS[name]
a = make_config_tensor(name)
A = torch.from_numpy(np.asfortranarray(a)).cuda()
fn = rt.rsthosvd if c["algo"] == "rsthosvd" else rt.rthosvd
dims = list(A.shape)
ranks = c["ranks"]
ws = torch.empty(rt.workspace_bytes(c["algo"] == "rsthosvd", dims, ranks, c["p"], c["q"]), dtype=torch.uint8,
                 device="cuda")
U = [torch.empty((r, n), device="cuda").t() for n, r in zip(dims, ranks)]
core = rt.as_column_major(torch.empty(ranks, device="cuda"))
args = (A, ranks, c["p"], c["q"], c["omega_seed"])
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(2):
        fn(*args, out=(core, U), workspace=ws)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
ref_core = core.clone()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    fn(*args, out=(core, U), workspace=ws)
core.zero_()
g.replay()
torch.cuda.synchronize()
same = torch.equal(core, ref_core)


def timed(f, reps=20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t_eager = timed(lambda: fn(*args, out=(core, U), workspace=ws))
t_graph = timed(g.replay)
print(f"{name}: graph replay bit-identical to eager: {same}; eager {t_eager:.3f} ms, graph {t_graph:.3f} ms")

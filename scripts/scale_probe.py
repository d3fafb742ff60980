"""Which kernel fails on a 1e15-scaled tensor (debugging): python scripts/scale_probe.py <scale>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_04840_b200 as rt  # noqa: E402
from workloads import CONFIGS, make_config_tensor  # noqa: E402

scale = float(sys.argv[1])
c = CONFIGS["c5"]
a = make_config_tensor("c5", dims=(600, 200, 150)) * scale
print("max|a|", np.abs(a).max(), flush=True)
A = torch.from_numpy(np.asfortranarray(a, dtype=np.float32)).cuda()
core, U, rep = rt.solve(A, (30, 20, 15), 8, 2, c["omega_seed"], sequential=True, report=True)
torch.cuda.synchronize()
print("ok", float(core.abs().max()), [float(u.abs().max()) for u in U], rep.alpha_trace[:3])

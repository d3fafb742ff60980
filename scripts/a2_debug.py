"""A.2 vs Alg. 4 alpha traces on the reduced C3 input, GPU vs oracle (diagnostics)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import tucker  # noqa: E402
from paper_2506_04840_b200 import rsthosvd, rsthosvd_a2  # noqa: E402
from tests.gpu_util import to_device_colmajor  # noqa: E402
from workloads import CONFIGS, make_config_tensor  # noqa: E402

c = CONFIGS["c3"]
a = make_config_tensor("c3", dims=(160, 150, 140))
A = to_device_colmajor(a, torch)
for name, gf, of in [("alg4", rsthosvd, tucker.rsthosvd), ("a2", rsthosvd_a2, tucker.rsthosvd_a2)]:
    o = of(a, c["ranks"], c["p"], c["q"], c["omega_seed"])
    for rep_i in range(2):
        _, _, rep = gf(A, c["ranks"], c["p"], c["q"], c["omega_seed"], report=True)
        torch.cuda.synchronize()
        for k in range(3):
            print(name, os.environ.get("RTK_PATH"), rep_i, k, np.round(rep.alpha_trace[k], 4), np.round(o.traces[k].alpha, 4),
                  "sigma_ll", np.round(o.traces[k].sigma_ll, 4))

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2506_04840_b200 as rt
from workloads import CONFIGS, make_config_tensor, make_config_tensor_torch
for name in sys.argv[1:]:
    c = CONFIGS[name]
    A = make_config_tensor_torch(name) if name == "c5" else torch.from_numpy(np.asfortranarray(make_config_tensor(name))).cuda()
    core, U, rep = rt.solve(A, c["ranks"], c["p"], c["q"], c["omega_seed"], sequential=c["algo"] == "rsthosvd", report=True)
    print(name, "sweeps(last step)", rep.jacobi_sweeps, "alpha", [round(a[-1], 6) for a in rep.alpha_trace], flush=True)

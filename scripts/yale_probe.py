"""Yale-B stand-in (480x640x560, q = 1): RE and alpha traces against the oracle on the fp16 pair engine
and with RTK_PAIR_F16=0 (3xTF32), to see which engine the 3.5e-7 RE difference of the context run comes from."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_04840_b200 as rt  # noqa: E402
from oracle import metrics, tucker  # noqa: E402
from workloads import CONFIGS, make_config_tensor  # noqa: E402
dims, ranks = (480, 640, 560), (50, 50, 50)
a = make_config_tensor("c5", dims=dims)
A = rt.as_column_major(torch.from_numpy(a).cuda())
orc = tucker.rsthosvd(a, ranks, 10, 1, 5002)
re_o = metrics.relative_error(a, orc.core, orc.factors)
gaps = metrics.mode_gaps(a, ranks, orc.factors, True)
print("oracle RE", re_o, "gaps", gaps)
for env in ({}, {"RTK_PAIR_F16": "0"}, {"RTK_PAIR": "0"}, {"RTK_FUSED": "0"}, {"RTK_PATH": "ffma"}):
    for k in ("RTK_PAIR_F16", "RTK_PATH", "RTK_PAIR", "RTK_FUSED"):
        os.environ.pop(k, None)
    os.environ.update(env)
    core, U, rep = rt.rsthosvd(A, ranks, 10, 1, 5002, report=True)
    torch.cuda.synchronize()
    gU = [u.cpu().numpy() for u in U]
    re_g = metrics.relative_error(a, core.cpu().numpy(), gU)
    ang = [metrics.max_principal_angle(uo, ug) for uo, ug in zip(orc.factors, gU)]
    # signed (gpu - oracle) / oracle of the (single, q = 1) alpha per mode: a negative value in every mode
    # on every tensor engine points at the round-toward-zero fp32 accumulation of the tensor core
    al = [float(((np.asarray(rep.alpha_trace[k]) - np.asarray(tr.alpha)) / (np.abs(np.asarray(tr.alpha)) + 1e-300))[0])
          for k, tr in enumerate(orc.traces)]
    print(env, "RE", re_g, "rel diff", abs(re_g - re_o) / re_o, "angles", ang, "alpha signed rel err", al, flush=True)

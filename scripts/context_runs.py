"""Optional context runs of SURVEY.md 8(d): shape-only stand-ins for the paper's real-data rows (Table 1,
PAPER.md:916-930; Yale B 480x640x560 ranks (50,50,50), COIL-100 1152x1024x300 ranks (30,30,15),
Washington DC Mall 1280x307x191 ranks (40,30,20)), oversampling 10, q = 1, Alg. 4.  The datasets are not
in this container: the tensors are filled with C5's recipe (low Tucker rank + noise, workloads/), so only
the GPU time is set beside the paper's CPU seconds (another machine: context, not a target) and RE is
compared with the float64 oracle on the same tensor, never with the paper's RE.

python scripts/context_runs.py > profiles/r2m_context_runs.md
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_04840_b200 as rt  # noqa: E402
from oracle import metrics, tucker  # noqa: E402
from workloads import CONFIGS, make_config_tensor  # noqa: E402

ROWS = [  # name, dims, ranks, paper's Alg. 4 CPU seconds (Table 1)
    ("Yale B", (480, 640, 560), (50, 50, 50), 0.86),
    ("COIL-100", (1152, 1024, 300), (30, 30, 15), 1.25),
    ("Washington DC", (1280, 307, 191), (40, 30, 20), 0.33),
]
P, Q, SEED = 10, 1, CONFIGS["c5"]["omega_seed"]

print("| stand-in for | shape | ranks | GPU ms / solve (median of 5, A in HBM) | HBM floor ms (3 passes over A) | "
      "RE GPU | RE oracle | rel. diff | orth | oracle s (CPU, %d cores) | paper's CPU s (its machine) |" % os.cpu_count())
print("|---|---|---|---|---|---|---|---|---|---|---|")
for name, dims, ranks, paper_s in ROWS:
    a = make_config_tensor("c5", dims=dims)
    A = torch.from_numpy(a).cuda()                    # Fortran-ordered host array -> column-major strides
    A = rt.as_column_major(A)
    for _ in range(4):
        out = rt.rsthosvd(A, ranks, P, Q, SEED)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = rt.rsthosvd(A, ranks, P, Q, SEED)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    core, U = out
    gU = [u.cpu().numpy() for u in U]
    re_g = metrics.relative_error(a, core.cpu().numpy(), gU)
    orth = max(metrics.orthonormality(u) for u in gU)
    del A
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    orc = tucker.rsthosvd(a, ranks, P, Q, SEED)
    t_or = time.perf_counter() - t0
    re_o = metrics.relative_error(a, orc.core, orc.factors)
    floor = 3 * a.size * 4 / 6537e9 * 1e3             # sketch + one power step + shrink of mode 1 dominate
    print(f"| {name} | {'x'.join(map(str, dims))} | {ranks} | {np.median(ts):.3f} | {floor:.3f} | {re_g:.6e} | "
          f"{re_o:.6e} | {abs(re_g - re_o) / re_o:.1e} | {orth:.1e} | {t_or:.2f} | {paper_s} |", flush=True)

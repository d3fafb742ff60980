"""Debug: Alg. A.2 with p = 0 on a matrix (GPU vs oracle per-mode angles / gaps)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_04840_b200 as rt  # noqa: E402
from oracle import metrics, tucker  # noqa: E402
from workloads import orthonormal_factor, tucker_tensor  # noqa: E402

for dims, ranks, p, q in [((34, 572), (5, 4), 0, 1), ((148, 656), (5, 3), 0, 3), ((34, 572), (5, 4), 1, 1)]:
    rng = np.random.default_rng(5)
    cr = [min(n, r + 3) for n, r in zip(dims, ranks)]
    core = rng.standard_normal(cr) * np.exp(-0.3 * np.indices(cr).sum(axis=0))
    a = tucker_tensor(core, [orthonormal_factor(n, r, rng) for n, r in zip(dims, cr)], noise=1e-3, rng=rng)
    A = torch.from_numpy(np.asfortranarray(a)).cuda()
    g_core, g_U = rt.rsthosvd_a2(A, ranks, p, q, 5)
    orc = tucker.rsthosvd_a2(a, ranks, p, q, 5)
    gU = [u.cpu().numpy() for u in g_U]
    gaps = metrics.mode_gaps(a, ranks, orc.factors, True)
    print(dims, ranks, p, q, "gaps", np.round(gaps, 3),
          "angles", [float(metrics.max_principal_angle(uo, ug)) for uo, ug in zip(orc.factors, gU)],
          "RE", metrics.relative_error(a, g_core.cpu().numpy(), gU), metrics.relative_error(a, orc.core, orc.factors))
    print(" core g", np.round(g_core.cpu().numpy()[:3, :3], 4).tolist(), " core o", np.round(orc.core[:3, :3], 4).tolist())

print("--- Alg. 4, same inputs")
for dims, ranks, p, q in [((34, 572), (5, 4), 0, 1), ((148, 656), (5, 3), 0, 3)]:
    rng = np.random.default_rng(5)
    cr = [min(n, r + 3) for n, r in zip(dims, ranks)]
    core = rng.standard_normal(cr) * np.exp(-0.3 * np.indices(cr).sum(axis=0))
    a = tucker_tensor(core, [orthonormal_factor(n, r, rng) for n, r in zip(dims, cr)], noise=1e-3, rng=rng)
    A = torch.from_numpy(np.asfortranarray(a)).cuda()
    g_core, g_U = rt.rsthosvd(A, ranks, p, q, 5)
    orc = tucker.rsthosvd(a, ranks, p, q, 5)
    gU = [u.cpu().numpy() for u in g_U]
    print(dims, ranks, p, q, "angles", [float(metrics.max_principal_angle(uo, ug)) for uo, ug in zip(orc.factors, gU)])
    # A.2 internals: oracle Q_1 vs GPU (via Alg. 4's U_1 with r = l)
    q1 = tucker._range_finder(tucker.unfold(a.astype(np.float64), 0), ranks[0], p, q, 5, 1, True, full=True)[0]
    print("   oracle Q1 vs GPU U1 (Alg.4) angle", float(metrics.max_principal_angle(q1, gU[0])))

"""Re-run one parity-sweep case by replaying the sweep RNG up to case index i (diagnostics)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import paper_2506_04840_b200 as rt  # noqa: E402
from oracle import metrics, tucker  # noqa: E402
from parity_sweep import case  # noqa: E402
from workloads import orthonormal_factor, tucker_tensor  # noqa: E402

seed, target = int(sys.argv[1]), sys.argv[2]
rng = np.random.default_rng(seed)
while True:
    c = case(rng)
    if c is None:
        continue
    dims, ranks = c["dims"], c["ranks"]
    cr = [min(n, r + 3) for n, r in zip(dims, ranks)]
    core = rng.standard_normal(cr) * np.exp(-0.3 * np.indices(cr).sum(axis=0))
    a = tucker_tensor(core, [orthonormal_factor(n, r, rng) for n, r in zip(dims, cr)], noise=1e-3, rng=rng)
    if str(c["dims"]) == target:
        break
print(c)
for path in ["ffma", "tc"]:
    os.environ["RTK_PATH"] = path
    A = torch.from_numpy(np.asfortranarray(a)).cuda()
    seq = c["algo"] != "t"
    g_core, g_U, rep = rt.solve(A, ranks, c["p"], c["q"], 5, sequential=seq, shift=c["shift"], report=True,
                                omega_kind=c.get("omega", 0))
    ofn = tucker.rsthosvd if seq else tucker.rthosvd
    orc = ofn(a, ranks, c["p"], c["q"], 5, shift=c["shift"], omega_kind=c.get("omega", 0))
    gU = [u.cpu().numpy() for u in g_U]
    gaps = metrics.mode_gaps(a, ranks, orc.factors, seq)
    print(path, "gaps", np.round(gaps, 4), "angles", [f"{metrics.max_principal_angle(uo, ug):.2e}" for uo, ug in zip(orc.factors, gU)])
    print("  RE", metrics.relative_error(a, g_core.cpu().numpy(), gU), metrics.relative_error(a, orc.core, orc.factors),
          "fallback", rep.fallback, "numeric", rep.numeric)
    for k, tr in enumerate(orc.traces):
        print("  mode", k + 1, "alpha gpu", np.round(rep.alpha_trace[k], 6), "orc", np.round(tr.alpha, 6),
              "sigma_ll", np.round(tr.sigma_ll, 6))
    for k in range(2):
        d = np.sum(gU[k].astype(np.float64) * orc.factors[k], axis=0)
        print("  mode", k + 1, "column cosines < 0.999:", [(j, round(float(x), 6)) for j, x in enumerate(d) if x < 0.999])

"""Tensor B at 600^3 through the GPU path: q_used / RE / numeric status for
Alg. 4 and Alg. B.1 (diagnostics; not product code)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2506_04840_b200 import solve  # noqa: E402
from workloads import make_tensor_b_torch, tensor_b_spectrum  # noqa: E402


def re_dev(A, core, U):
    a = A.double()
    rec = core.double()
    for k, u in enumerate(U):
        rec = torch.tensordot(rec, u.double(), dims=([0], [1]))   # cycles modes
    return float(torch.linalg.vector_norm(a - rec) / torch.linalg.vector_norm(a))


for kind in sys.argv[1:] or ["slow", "fast"]:
    A = make_tensor_b_torch(600, kind, 11)
    v = tensor_b_spectrum(600, kind)
    for r in (20, 40):
        cf = np.sqrt(np.sum(v[r:] ** 2) / np.sum(v ** 2))
        for tol in (0.0, 0.5, 0.1, 0.05, 0.01):
            q = 3 if tol == 0.0 else 30
            core, U, rep = solve(A, (r, r, r), 10, q, 5, sequential=True, report=True, pve_tol=tol)
            torch.cuda.synchronize()
            print(f"{kind} r={r} tol={tol}: q_used={rep.q_used} numeric={rep.numeric} "
                  f"fallback={rep.fallback} RE={re_dev(A, core, U):.5e} closed form {cf:.5e}", flush=True)

"""A/B check of two kernel paths on one config (GPU only, no oracle): runs the solve with env
RTK_FUSED=0 and =1 and compares factors (principal angles) and RE computed on the GPU in fp64.

python scripts/ab_paths.py c5
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2506_04840_b200 as rt  # noqa: E402
from workloads import CONFIGS, make_config_tensor_torch  # noqa: E402


def re_gpu(A, core, U):
    # ||A - core x_1 U_1 ... x_d U_d||_F / ||A||_F in fp64, slab by slab over the last mode
    d = A.dim()
    g = core.double()
    for k in range(d - 1):
        g = torch.movedim(torch.tensordot(U[k].double(), g, dims=([1], [k])), 0, k)
    Ud = U[-1].double()
    num = 0.0
    den = 0.0
    nd = A.shape[-1]
    for s0 in range(0, nd, 50):
        s1 = min(nd, s0 + 50)
        slab = A[..., s0:s1].double()
        rec = torch.tensordot(g, Ud[s0:s1], dims=([d - 1], [1]))
        num += float(((slab - rec) ** 2).sum())
        den += float((slab ** 2).sum())
    return (num / den) ** 0.5


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    c = CONFIGS[name]
    A = make_config_tensor_torch(name)
    out = {}
    for flag in ("0", "1"):
        os.environ["RTK_FUSED"] = flag
        core, U, rep = rt.solve(A, c["ranks"], c["p"], c["q"], c["omega_seed"],
                                sequential=c["algo"] == "rsthosvd", report=True)
        torch.cuda.synchronize()
        out[flag] = (core.clone(), [u.clone() for u in U], rep)
        print(f"RTK_FUSED={flag}: RE {re_gpu(A, core, U):.9e} alpha {[round(t[-1], 6) for t in rep.alpha_trace]}",
              flush=True)
    for k in range(len(c["dims"])):
        u0, u1 = out["0"][1][k].double(), out["1"][1][k].double()
        s = torch.linalg.svdvals(u0.T @ u1)
        ang = float(torch.arccos(torch.clamp(s.min(), max=1.0)))
        orth = float(torch.linalg.norm(u1.T @ u1 - torch.eye(u1.shape[1], dtype=torch.float64, device=u1.device)))
        print(f"mode {k+1}: max principal angle {ang:.3e}  orth(fused) {orth:.2e}")


if __name__ == "__main__":
    main()

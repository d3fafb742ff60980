"""Small solves through the public API for compute-sanitizer (memcheck / racecheck / synccheck):
C1 (Alg. 3, strided FFMA views + tcgen05 mode 1), a 2-CTA fused-engine case (n_1 = 640 > 512, incl.
the fused Omega-plane sketch forced on), Alg. A.2 and Alg. B.1.  Each case is also checked against
the float64 oracle's RE so that a sanitizer-perturbed run that computes garbage is visible.

python scripts/sanitize_cases.py [case ...]   (default: all)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2506_04840_b200 as rt  # noqa: E402
from oracle import metrics, tucker  # noqa: E402
from workloads import CONFIGS, make_config_tensor, orthonormal_factor, tucker_tensor  # noqa: E402


def dev(a):
    return torch.from_numpy(np.asfortranarray(a, dtype=np.float32)).cuda()


def check(name, a, core, U, orc):
    torch.cuda.synchronize()
    re_g = metrics.relative_error(a, core.cpu().numpy(), [u.cpu().numpy() for u in U])
    re_o = metrics.relative_error(a, orc.core, orc.factors)
    ok = abs(re_g - re_o) <= 1e-4 * re_o + 1e-7
    print(f"{name}: RE gpu {re_g:.6e} oracle {re_o:.6e} {'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def case_c1():
    c = CONFIGS["c1"]
    a = make_config_tensor("c1")
    core, U = rt.rthosvd(dev(a), c["ranks"], c["p"], c["q"], c["omega_seed"])
    return check("c1 (Alg. 3)", a, core, U, tucker.rthosvd(a, c["ranks"], c["p"], c["q"], c["omega_seed"]))


def _tensor(dims, ranks, seed):
    rng = np.random.default_rng(seed)
    cr = tuple(min(n, r + 3) for n, r in zip(dims, ranks))
    core = rng.standard_normal(cr) * np.exp(-0.3 * np.indices(cr).sum(axis=0))
    return tucker_tensor(core, [orthonormal_factor(n, r, rng) for n, r in zip(dims, cr)], noise=1e-3, rng=rng)


def case_fused2cta():
    dims, ranks = (640, 40, 36), (20, 8, 6)
    a = _tensor(dims, ranks, 640)
    os.environ["RTK_FUSED_SKETCH_MIN"] = "0"
    core, U = rt.rsthosvd(dev(a), ranks, 6, 3, 77)
    os.environ.pop("RTK_FUSED_SKETCH_MIN")
    return check("640x40x36 (Alg. 4, 2-CTA fused engine + fused sketch)", a, core, U,
                 tucker.rsthosvd(a, ranks, 6, 3, 77))


def case_a2():
    dims, ranks = (96, 40, 36), (12, 6, 5)
    a = _tensor(dims, ranks, 96)
    core, U = rt.rsthosvd_a2(dev(a), ranks, 4, 2, 17)
    return check("96x40x36 (Alg. A.2)", a, core, U, tucker.rsthosvd_a2(a, ranks, 4, 2, 17))


def case_b1():
    dims, ranks = (60, 50, 40), (6, 5, 4)
    a = _tensor(dims, ranks, 60)
    core, U = rt.solve(dev(a), ranks, 4, 8, 21, sequential=True, pve_tol=3e-2)
    return check("60x50x40 (Alg. B.1, tol 3e-2)", a, core, U, tucker.rsthosvd(a, ranks, 4, 0, 21, pve=(3e-2, 8)))


CASES = {"c1": case_c1, "fused2cta": case_fused2cta, "a2": case_a2, "b1": case_b1}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    ok = all([CASES[n]() for n in names])
    sys.exit(0 if ok else 1)

"""Randomised GPU-vs-oracle parity sweep (robustness, not a unit test): random shapes, ranks, p, q,
algorithm (Alg. 3 / 4 / A.2), streaming path, shift on/off and sketch type, each checked with the
north_star tolerances.  Prints one line per case and a summary; exits 1 on any failure.

python scripts/parity_sweep.py [n_cases] [seed] [big]
"big": d = 3 with n_1 in [257, 1000] and up to 2e7 entries, tensor path only, so mode 1 (and often mode 2)
runs on the CTA-pair engine (fp16 power steps, pair sketch / shrink), the fused sketch forced on at random.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_04840_b200 as rt  # noqa: E402
from oracle import metrics, tucker  # noqa: E402
from workloads import orthonormal_factor, tucker_tensor  # noqa: E402


def case(rng, big=False):
    d = 3 if big else int(rng.integers(2, 5))
    budget = 20000000 if big else {2: 400000, 3: 2000000, 4: 1500000}[d]
    while True:
        if big:
            dims = [int(rng.integers(257, 1001)), int(rng.integers(8, 400)), int(rng.integers(8, 400))]
            if rng.integers(0, 4) == 0:          # sometimes the long mode is not the first
                dims = [dims[1], dims[0], dims[2]]
        else:
            dims = [int(rng.integers(2, 700 if d == 2 else (220 if d == 3 else 48))) for _ in range(d)]
        if int(np.prod(dims)) <= budget:
            break
    algo = ["t", "st", "a2"][int(rng.integers(0, 3))] if d > 1 else "st"
    p = int(rng.integers(0, 11))
    ranks = []
    for k, n in enumerate(dims):
        ranks.append(int(rng.integers(1, max(2, min(n, 56 if big else 40)))))
    # respect l_k <= min(n_k, m_k) (m_k over the shrunk extents for ST / A.2)
    for _ in range(50):
        ok = True
        keep = []
        for k, n in enumerate(dims):
            l = ranks[k] + p
            m = 1
            for j, nj in enumerate(dims):
                if j == k:
                    continue
                if algo != "t" and j < k:
                    m *= keep[j]
                else:
                    m *= nj
            if l > n or l > m or l > (64 if algo == "a2" else 96):
                ok = False
                if p > 0:
                    p -= 1
                else:
                    ranks[k] = max(1, ranks[k] // 2)
                break
            keep.append(ranks[k] + (p if algo == "a2" else 0))
        if ok:
            break
    else:
        return None
    q = int(rng.integers(1, 5))
    path = "tc" if big else ["ffma", "tc"][int(rng.integers(0, 2))]
    shift = bool(rng.integers(0, 4) > 0)
    omega = int(rng.integers(0, 4)) if rng.integers(0, 3) == 0 else 0
    c = dict(dims=dims, ranks=ranks, p=p, q=q, algo=algo, path=path, shift=shift, omega=omega)
    if big:
        c["fused_sketch_min"] = 0 if rng.integers(0, 2) else None
    return c


def main():
    n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
    big = len(sys.argv) > 3 and sys.argv[3] == "big"
    fails = 0
    ties = 0
    done = 0
    while done < n_cases:
        c = case(rng, big)
        if c is None:
            continue
        done += 1
        dims, ranks = c["dims"], c["ranks"]
        cr = [min(n, r + 3) for n, r in zip(dims, ranks)]
        core = rng.standard_normal(cr) * np.exp(-0.3 * np.indices(cr).sum(axis=0))
        a = tucker_tensor(core, [orthonormal_factor(n, r, rng) for n, r in zip(dims, cr)], noise=1e-3, rng=rng)
        os.environ["RTK_PATH"] = c["path"]
        if c.get("fused_sketch_min") is not None:
            os.environ["RTK_FUSED_SKETCH_MIN"] = str(c["fused_sketch_min"])
        else:
            os.environ.pop("RTK_FUSED_SKETCH_MIN", None)
        A = torch.from_numpy(np.asfortranarray(a)).cuda()
        seq, variant = c["algo"] != "t", 1 if c["algo"] == "a2" else 0
        try:
            g_core, g_U = rt.solve(A, ranks, c["p"], c["q"], 5, sequential=seq, variant=variant, shift=c["shift"],
                                   omega_kind=c["omega"])
            torch.cuda.synchronize()
        except Exception as e:   # noqa: BLE001
            print("ERROR", c, e, flush=True)
            fails += 1
            continue
        fn = {"t": tucker.rthosvd, "st": tucker.rsthosvd, "a2": tucker.rsthosvd_a2}[c["algo"]]
        orc = fn(a, ranks, c["p"], c["q"], 5, shift=c["shift"], omega_kind=c["omega"])
        gU = [u.cpu().numpy() for u in g_U]
        re_g = metrics.relative_error(a, g_core.cpu().numpy(), gU)
        re_o = metrics.relative_error(a, orc.core, orc.factors)
        gaps = list(metrics.mode_gaps(a, ranks, orc.factors, seq))
        if c["algo"] == "a2":   # U_k is unique only up to the l-core unfolding's column count
            ls = [r + c["p"] for r in ranks]
            for k in range(len(dims)):
                cols = int(np.prod(ranks[:k]) * np.prod(ls[k + 1:]))
                if ranks[k] > cols:
                    gaps[k] = 0.0   # null-space completion: any orthonormal choice is valid
        orth = max(metrics.orthonormality(u) for u in gU)

        def check(o):
            re_o = metrics.relative_error(a, o.core, o.factors)
            ang = max([metrics.max_principal_angle(uo, ug) for uo, ug, gp in zip(o.factors, gU, gaps) if gp > 0.1]
                      or [0.0])
            return abs(re_g - re_o) <= 1e-4 * re_o + 1e-7 and orth <= 1e-5 and ang <= 1e-3, re_o, ang

        ok, re_o, ang = check(orc)
        tag = "ok  " if ok else "FAIL"
        if not ok and c["algo"] == "st":
            # C6's residual risk: a column of an earlier U_k whose sign pivot is not determined at
            # the precision of the data (top-two |entries| closer than the column's own GPU/oracle
            # difference) may carry the other sign on the GPU; ST then feeds that sign to every later
            # mode, which then draws effectively different sketches.  Such a case is reported as
            # undetermined, never re-run with a GPU-chosen sign: only what the sign cannot change is
            # compared (orthonormality everywhere, principal angles of modes up to the ambiguous one).
            k_amb = None
            for k in range(len(dims) - 1):
                uo, ug = orc.factors[k], gU[k].astype(np.float64)
                for j in range(uo.shape[1]):
                    if float(np.dot(uo[:, j], ug[:, j])) < -0.99:
                        col = np.sort(np.abs(uo[:, j]))[::-1]
                        if col.size > 1 and (col[0] - col[1]) <= 20 * (float(np.max(np.abs(uo[:, j] + ug[:, j])))
                                                                       + 1e-5 * col[0]):
                            k_amb = k if k_amb is None else min(k_amb, k)
            if k_amb is not None:
                ang = max([metrics.max_principal_angle(uo, ug)
                           for kk, (uo, ug, gp) in enumerate(zip(orc.factors, gU, gaps)) if kk <= k_amb and gp > 0.1]
                          or [0.0])
                ok = orth <= 1e-5 and ang <= 1e-3
                tag = "UNDET" if ok else "FAIL"
                ties += 1 if ok else 0
        fails += 0 if ok else 1
        print(tag, c, f"RE {re_g:.6e}/{re_o:.6e} orth {orth:.1e} angle {ang:.1e}", flush=True)
    print(f"{done - fails}/{done} cases within tolerance ({ties} with an undetermined sign pivot, C6: "
          "sign-invariant checks only)")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()

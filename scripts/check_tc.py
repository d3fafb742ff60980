"""Quick GPU check of the tcgen05 power step vs fp64 (and vs the FFMA path)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2506_04840_b200 as rt
shapes = [(64, 4096, 10), (200, 3000, 30), (400, 2001, 40), (1000, 1234, 60), (37, 333, 13), (1000, 200000, 60), (80, 5000, 15)]
for n, m, l in shapes:
    rng = np.random.default_rng(n + m)
    M = rng.standard_normal((n, m)).astype(np.float32)
    Q = np.linalg.qr(rng.standard_normal((n, l)))[0].astype(np.float32)
    Md = torch.from_numpy(np.asfortranarray(M)).cuda()
    Qd = torch.from_numpy(Q).cuda()
    ref = M.astype(np.float64) @ (M.astype(np.float64).T @ Q.astype(np.float64))
    for path in ["tc", "ffma"]:
        os.environ["RTK_PATH"] = path
        Y = rt.power_step(Md, Qd)
        torch.cuda.synchronize()
        t0 = time.time(); reps = 3
        for _ in range(reps): rt.power_step(Md, Qd)
        torch.cuda.synchronize(); dt = (time.time() - t0) / reps
        Yn = Y.cpu().numpy()
        err = np.linalg.norm(Yn - ref) / np.linalg.norm(ref)
        print(f"n={n} m={m} l={l} path={path}: rel err {err:.2e}  ({dt*1e3:.2f} ms incl. alloc)", flush=True)

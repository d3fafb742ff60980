"""Bisect the fp16 pair engine failure: back-to-back power steps and a solve, with PDL on/off."""
import os
import subprocess
import sys

PS = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2506_04840_b200 as rt
n, m, l, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
g = torch.Generator(device="cuda"); g.manual_seed(0)
M = torch.randn((m, n), device="cuda", generator=g).t()
Q = torch.linalg.qr(torch.randn((n, l), device="cuda", generator=g, dtype=torch.float64))[0].float()
for _ in range(reps):
    Y = rt.power_step(M, Q)
torch.cuda.synchronize()
print("ok", float(Y.norm()))
'''
SOLVE = r'''
import sys, torch
sys.path.insert(0, ".")
import paper_2506_04840_b200 as rt
from workloads import CONFIGS, make_config_tensor_torch
name = sys.argv[1]
c = CONFIGS[name]
A = make_config_tensor_torch(name) if len(sys.argv) < 3 else torch.randn(tuple(int(x) for x in sys.argv[2].split("x")), device="cuda").t().contiguous().t()
core, U = rt.rsthosvd(A, c["ranks"], c["p"], c["q"], c["omega_seed"])
torch.cuda.synchronize()
print("ok", float(core.norm()))
'''
cases = [("ps", ["1000", "1000000", "60", "2"], {}), ("ps", ["1000", "1000000", "60", "2"], {"RTK_PDL": "0"}),
         ("ps", ["1000", "200000", "60", "6"], {}),
         ("solve", ["c5"], {}), ("solve", ["c5"], {"RTK_PDL": "0"}), ("solve", ["c5"], {"CUDA_LAUNCH_BLOCKING": "1"}),
         ("solve", ["c3"], {}), ("solve", ["c5"], {"RTK_PAIR_SHRINK": "0"})]
for kind, args, env in cases:
    e = {**os.environ, "RTK_POWER_F16": "1", **env}
    try:
        r = subprocess.run([sys.executable, "-c", PS if kind == "ps" else SOLVE, *args], capture_output=True,
                           text=True, timeout=120, env=e)
        out = (r.stdout.strip().splitlines() or [""])[-1]
        err = (r.stderr.strip().splitlines() or [""])[-1]
        print(kind, args, env, "rc", r.returncode, out, err[-300:], flush=True)
    except subprocess.TimeoutExpired:
        print(kind, args, env, "TIMEOUT", flush=True)

"""Probe the fp16 pair power step across unfolding widths (subprocess per case, with a timeout):
python scripts/f16_probe.py"""
import subprocess
import sys

CODE = r'''
import sys, torch, numpy as np
sys.path.insert(0, ".")
import paper_2506_04840_b200 as rt
n, m, l = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
g = torch.Generator(device="cuda"); g.manual_seed(0)
M = torch.randn((m, n), device="cuda", generator=g).t()
Q = torch.linalg.qr(torch.randn((n, l), device="cuda", generator=g, dtype=torch.float64))[0].float()
Y = rt.power_step(M, Q); torch.cuda.synchronize()
ref = (M.double() @ (M.double().t() @ Q.double()))
print("err", float((Y.double() - ref).norm() / ref.norm()))
'''
for n, m, l in [(1000, 200000, 60), (1000, 300000, 60), (1000, 400000, 60), (1000, 600000, 60),
                (1000, 1000000, 60), (1000, 50000, 60), (400, 160000, 40)]:
    try:
        r = subprocess.run([sys.executable, "-c", CODE, str(n), str(m), str(l)], capture_output=True, text=True,
                           timeout=60, env={**__import__("os").environ, "RTK_POWER_F16": "1"})
        out = (r.stdout.strip().splitlines() or [""])[-1]
        err = (r.stderr.strip().splitlines() or [""])[-1]
        print(n, m, l, "rc", r.returncode, out, err[-200:], flush=True)
    except subprocess.TimeoutExpired:
        print(n, m, l, "TIMEOUT", flush=True)

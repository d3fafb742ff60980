"""Sweep tile plans for the fused power step on one shape (GPU).

python scripts/tune_tile.py n m l  "R,TC,NCG,b" ...
Prints ms per launch (CUDA events) and achieved FP32 TFLOP/s for each plan.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, json, torch
sys.path.insert(0, ROOT)
import paper_2506_04840_b200 as rt
n, m, l = map(int, sys.argv[1:4])
g = torch.Generator(device="cuda"); g.manual_seed(0)
M = torch.randn((m, n), device="cuda", generator=g).t()        # column-major n x m
Q = torch.linalg.qr(torch.randn((n, l), device="cuda", generator=g, dtype=torch.float64))[0].float()
for _ in range(2): rt.power_step(M, Q)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
rt.profile_begin()
e0.record()
for _ in range(reps): rt.power_step(M, Q)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(json.dumps({"plan": os.environ.get("RTK_PLAN_POWER", "auto"), "ms": ms,
                  "tflops": 4.0 * n * m * l / ms / 1e9}))
'''.replace("ROOT", repr(ROOT))


def main():
    n, m, l = sys.argv[1:4]
    plans = sys.argv[4:] or ["auto"]
    for p in plans:
        env = dict(os.environ)
        if p != "auto":
            env["RTK_PLAN_POWER"] = p
        env["RTK_VERBOSE"] = "1"
        r = subprocess.run([sys.executable, "-c", CHILD, n, m, l], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr.strip()[-500:], flush=True)
        plan_lines = [x for x in r.stderr.splitlines() if "[rtk] plan" in x]
        if plan_lines:
            print("   ", plan_lines[0], flush=True)


if __name__ == "__main__":
    main()

"""Per-l decision table, FP32 FFMA tiles vs the 3xTF32 tcgen05 fused engine (north_star: decide per
l from achieved HBM GB/s and FP32 / tensor-pipe utilisation).  One power step Y = M M^T Q of an
n x m column-major matrix through the rtk_power_step hook, timed with CUDA events (mean of reps).

python scripts/per_l_table.py [n] [m] [reps]        (ncu pipe metrics: scripts/per_l_ncu.sh)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2506_04840_b200 as rt  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
m = int(sys.argv[2]) if len(sys.argv) > 2 else 250000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
hbm = peaks["hbm_gbs"]
g = torch.Generator(device="cuda")
g.manual_seed(0)
M = torch.randn((m, n), device="cuda", generator=g).t()
rows = []
for l in (10, 15, 30, 40, 60, 80):
    Q = torch.linalg.qr(torch.randn((n, l), device="cuda", generator=g, dtype=torch.float64))[0].float()
    for path in ("ffma", "tc"):
        if path == "tc" and l > 64:
            rows.append((l, path, None))
            continue
        os.environ["RTK_PATH"] = path
        rt.power_step(M, Q)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            rt.power_step(M, Q)
        e1.record()
        torch.cuda.synchronize()
        rows.append((l, path, e0.elapsed_time(e1) / reps))
print(f"power step Y = M M^T Q, n = {n}, m = {m} ({4 * n * m / 1e9:.2f} GB), mean of {reps} (test hook incl. split/reduce)")
print("| l | path | ms | HBM GB/s (alg.) | frac of HBM | fp32-equivalent TFLOP/s |")
print("|---|---|---|---|---|---|")
for l, path, ms in rows:
    if ms is None:
        print(f"| {l} | tc | n/a (l > 64) | | | |")
        continue
    gbs = 4.0 * n * m / (ms * 1e-3) / 1e9
    tf = 4.0 * n * m * l / (ms * 1e-3) / 1e12
    print(f"| {l} | {path} | {ms:.3f} | {gbs:.0f} | {gbs / hbm:.2f} | {tf:.1f} |")

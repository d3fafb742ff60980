"""Signed error of one power step Y = M (M^T Q) on all-positive operands (no cancellation, so a rounding
bias cannot average out) against float64, per engine: a negative mean on the tcgen05 engines and ~0 on the
FFMA tiles is the round-toward-zero fp32 accumulator of the tensor core (DESIGN.md section 7 note,
profiles/r2m_context_runs.md).  python scripts/rz_probe.py"""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_04840_b200 as rt  # noqa: E402
from paper_2506_04840_b200 import _lib  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(7)
print("| n | m | l | engine | mean (Y - Y64) / Y64 | max abs rel |")
print("|---|---|---|---|---|---|")
for n, m, l in ((512, 200000, 60), (1000, 400000, 60)):
    M = torch.randn((m, n), generator=g, device="cuda", dtype=torch.float32).abs_().t()   # column-major n x m
    Q = torch.randn((n, l), generator=g, device="cuda", dtype=torch.float32).abs_() / n ** 0.5
    M64, Q64 = M.double(), Q.double()
    Y64 = M64 @ (M64.t() @ Q64)
    for name, env in (("3xTF32 pair", {}), ("fp16 pair", {"RTK_POWER_F16": "1"}), ("one-CTA fused", {"RTK_PAIR": "0"}),
                      ("two-kernel tcgen05", {"RTK_FUSED": "0"}), ("FFMA tiles", {"RTK_PATH": "ffma"})):
        for k in ("RTK_POWER_F16", "RTK_PAIR", "RTK_FUSED", "RTK_PATH"):
            os.environ.pop(k, None)
        os.environ.update(env)
        Y = _lib.power_step(M, Q)
        torch.cuda.synchronize()
        rel = (Y - Y64) / Y64
        print(f"| {n} | {m} | {l} | {name} | {rel.mean().item():+.3e} | {rel.abs().max().item():.3e} |", flush=True)

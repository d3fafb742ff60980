"""Run the fused power step a few times on an n x m column-major matrix (for ncu); prints the mean time
of the rtk_power_step test hook (fused kernel + its plane split and partial reduction)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_04840_b200 as rt  # noqa: E402

n, m, l = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
g = torch.Generator(device="cuda")
g.manual_seed(0)
M = torch.randn((m, n), device="cuda", generator=g).t()
Q = torch.linalg.qr(torch.randn((n, l), device="cuda", generator=g, dtype=torch.float64))[0].float()
rt.power_step(M, Q)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    rt.power_step(M, Q)
e1.record()
torch.cuda.synchronize()
print(f"ok: {e0.elapsed_time(e1) / reps:.3f} ms per power_step call (incl. the test hook's planes / reduction)")

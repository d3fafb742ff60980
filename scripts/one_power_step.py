"""Run the fused power step a few times on an n x m column-major matrix (for ncu)."""
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
for _ in range(reps):
    rt.power_step(M, Q)
torch.cuda.synchronize()
print("ok")

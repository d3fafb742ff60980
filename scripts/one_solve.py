"""One solve of a config through the public API (for ncu -s/-c launch selection)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_04840_b200 as rt  # noqa: E402
from workloads import CONFIGS, make_config_tensor_torch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
c = CONFIGS[name]
A = make_config_tensor_torch(name)
fn = rt.rsthosvd if c["algo"] == "rsthosvd" else rt.rthosvd
fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"])
torch.cuda.synchronize()
print("ok")

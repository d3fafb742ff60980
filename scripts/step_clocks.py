"""Phase clock counts of the cluster small solver (rtk_debug_step_clocks) for one config.

python scripts/step_clocks.py c5
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2506_04840_b200 as rt  # noqa: E402
from workloads import CONFIGS, make_config_tensor_torch  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
c = CONFIGS[name]
A = make_config_tensor_torch(name)
fn = rt.rsthosvd if c["algo"] == "rsthosvd" else rt.rthosvd
buf = torch.zeros(8 * 8 * 16, dtype=torch.float64, device="cuda")
lib = rt.load_library()
fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"])
lib.rtk_debug_step_clocks(ctypes.c_void_p(buf.data_ptr()))
fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"])
torch.cuda.synchronize()
lib.rtk_debug_step_clocks(None)
b = buf.view(8, 8, 16).cpu().numpy()
for k in range(len(c["dims"])):
    for s in range(c["q"] + 1):
        row = b[k, s]
        nt = int(row[0])
        print(f"mode {k+1} step {s}: eig={int(row[1])} two_pass={int(row[2])} phases(kcyc)=",
              [round(x / 1e3, 1) for x in row[3:3 + nt - 1]])

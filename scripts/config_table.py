"""All BASELINE configs on the GPU (device ms per solve, RE) beside the float64 oracle (CPU seconds,
RE) -- the evidence table behind DESIGN.md section 7.  C5's oracle runs on the host copy of the very
tensor the GPU solved (~20 GB of host RAM).

python scripts/config_table.py > profiles/r2_configs.md
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_04840_b200 as rt  # noqa: E402
from oracle import metrics, tucker  # noqa: E402
from workloads import CONFIGS, make_config_tensor, make_config_tensor_torch  # noqa: E402


def gpu_time(fn, A, c, reps=5, **kw):
    """Per call, synchronised (host enqueue latency included), after 4 warm-up calls: every call
    allocates new outputs, so two output sets alternate and both keys are captured as CUDA graphs
    before timing (rtk_api.cu solve_entry); then the back-to-back device time of 10 calls with the
    graph replay and with RTK_GRAPH=0 (direct enqueue)."""
    for _ in range(4):
        out = fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"], **kw)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"], **kw)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    b2b = {}
    for mode in ("graph", "direct"):
        if mode == "direct":
            os.environ["RTK_GRAPH"] = "0"
        core, U = out
        for _ in range(3):
            fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"], out=(core, U), **kw)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"], out=(core, U), **kw)
        e1.record()
        torch.cuda.synchronize()
        b2b[mode] = e0.elapsed_time(e1) / 10
        os.environ.pop("RTK_GRAPH", None)
    return float(np.median(ts)), b2b, out


print("| config | algorithm | GPU ms / solve (per call, synced, median of 5) | back-to-back ms (graph / direct) | RE GPU | RE oracle | rel. diff | oracle s (CPU, %d cores) |"
      % os.cpu_count())
print("|---|---|---|---|---|---|---|---|")
for name, c in CONFIGS.items():
    seq = c["algo"] == "rsthosvd"
    variants = [("Alg. 4" if seq else "Alg. 3", rt.rsthosvd if seq else rt.rthosvd,
                 tucker.rsthosvd if seq else tucker.rthosvd, {})]
    if seq and name != "c5":
        variants.append(("Alg. A.2", rt.rsthosvd_a2, tucker.rsthosvd_a2, {}))
    if name == "c5":
        A = make_config_tensor_torch(name)
        a = None
    else:
        a = make_config_tensor(name)
        A = torch.from_numpy(np.asfortranarray(a)).to("cuda")
    for label, gfn, ofn, kw in variants:
        ms, b2b, (core, U) = gpu_time(gfn, A, c, **kw)
        if a is None:
            a = A.cpu().numpy()
        re_g = metrics.relative_error(a, core.cpu().numpy(), [u.cpu().numpy() for u in U])
        t0 = time.perf_counter()
        orc = ofn(a, c["ranks"], c["p"], c["q"], c["omega_seed"])
        t_o = time.perf_counter() - t0
        re_o = metrics.relative_error(a, orc.core, orc.factors)
        print(f"| {name} | {label} | {ms:.3f} | {b2b['graph']:.3f} / {b2b['direct']:.3f} | {re_g:.6e} | {re_o:.6e} | {abs(re_g - re_o) / re_o:.1e} | {t_o:.2f} |",
              flush=True)

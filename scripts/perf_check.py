"""Performance regression check: device ms per solve of every config (median of 5) against the
stored round baseline (profiles/perf_baseline.json); prints a table and exits 1 if any config is
more than --tol (default 10 %) slower.  --update rewrites the baseline.

python scripts/perf_check.py [--tol 0.1] [--update]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_04840_b200 as rt  # noqa: E402
from workloads import CONFIGS, make_config_tensor, make_config_tensor_torch  # noqa: E402

BASE = os.path.join(ROOT, "profiles", "perf_baseline.json")


def median_ms(fn, args, reps=5):
    fn(*args)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(*args)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tol", type=float, default=0.10)
    ap.add_argument("--update", action="store_true")
    a = ap.parse_args()
    cur = {}
    for name, c in CONFIGS.items():
        A = (make_config_tensor_torch(name) if name == "c5"
             else torch.from_numpy(np.asfortranarray(make_config_tensor(name))).cuda())
        fn = rt.rsthosvd if c["algo"] == "rsthosvd" else rt.rthosvd
        cur[name] = median_ms(fn, (A, c["ranks"], c["p"], c["q"], c["omega_seed"]))
        del A
    base = json.load(open(BASE)) if os.path.exists(BASE) else {}
    bad = False
    for name, ms in cur.items():
        b = base.get(name)
        flag = ""
        if b is not None and ms > b * (1 + a.tol):
            flag, bad = "  SLOWER", True
        print(f"{name}: {ms:8.3f} ms   baseline {b if b is not None else float('nan'):8.3f}{flag}")
    if a.update:
        json.dump(cur, open(BASE, "w"), indent=1)
    sys.exit(1 if bad and not a.update else 0)


if __name__ == "__main__":
    main()

"""Is a solve bound by host launch overhead?  Device time of the public-API solve enqueued
directly (profiling off) against the same solve captured once in a CUDA graph and replayed.

python scripts/graph_probe.py [c4] [reps]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2506_04840_b200 as rt  # noqa: E402
from workloads import CONFIGS, make_config_tensor_torch  # noqa: E402


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    c = CONFIGS[name]
    A = make_config_tensor_torch(name)
    fn = rt.rsthosvd if c["algo"] == "rsthosvd" else rt.rthosvd
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        core, U = fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"])
    torch.cuda.synchronize()
    out = (core, U)

    def direct():
        fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"], out=out)

    with torch.cuda.stream(s):
        for _ in range(3):
            direct()
    torch.cuda.synchronize()
    t_direct = timed(direct, reps)
    import time
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    for _ in range(reps):
        direct()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    res = {"config": name, "direct_ms": round(t_direct, 4), "host_enqueue_ms": round((h1 - h0) * 1e3 / reps, 4)}
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=s):
            direct()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        res["graph_ms"] = round(timed(g.replay, reps), 4)
        ref = fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"])
        g.replay()
        torch.cuda.synchronize()
        res["graph_matches_direct"] = bool(torch.equal(out[0], ref[0]))
    except Exception as e:  # noqa: BLE001
        res["graph_error"] = repr(e)[:300]
    print(json.dumps(res))


if __name__ == "__main__":
    main()

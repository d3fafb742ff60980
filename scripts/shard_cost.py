"""Device ms of rtk_rsthosvd_shard with world = 1 (the whole tensor as one slab, identity
all-reduce) against rtk_rsthosvd on a config: the cost of the shard code path itself (Omega_k
materialised per mode, Y written before and its Gram read after the all-reduce point, the mode-d
gather).  python scripts/shard_cost.py [c5] [reps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2506_04840_b200 as rt  # noqa: E402
from workloads import CONFIGS, make_config_tensor_torch  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


name = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
c = CONFIGS[name]
A = make_config_tensor_torch(name)
dims = list(A.shape)
args = (c["ranks"], c["p"], c["q"], c["omega_seed"])
t_plain = timed(lambda: rt.rsthosvd(A, *args), reps)
t_shard = timed(lambda: rt.rsthosvd_shard(A, dims, 0, *args, allreduce=lambda t: None, root=True), reps)
c1, u1 = rt.rsthosvd(A, *args)
c2, u2 = rt.rsthosvd_shard(A, dims, 0, *args, allreduce=lambda t: None, root=True)
print(json.dumps({"config": name, "plain_ms": round(t_plain, 3), "shard_world1_ms": round(t_shard, 3),
                  "max_core_rel_diff": float((c1 - c2).abs().max() / c1.abs().max())}))

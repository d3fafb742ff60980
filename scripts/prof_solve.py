"""One profiled solve of a config through the public API; prints device ms by (kind, mode).

python scripts/prof_solve.py [c5] [reps] [a2|-] [omega_kind]
  a2: Alg. A.2 instead of the config's algorithm; omega_kind: 0 Gaussian, 1 uniform, 2/3 Khatri-Rao
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2506_04840_b200 as rt  # noqa: E402
from workloads import CONFIGS, make_config_tensor_torch  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    c = CONFIGS[name]
    A = make_config_tensor_torch(name)
    fn = rt.rsthosvd if c["algo"] == "rsthosvd" else rt.rthosvd
    if len(sys.argv) > 3 and sys.argv[3] == "a2":
        fn, name = rt.rsthosvd_a2, name + "-a2"
    kind = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    if kind:
        import functools
        fn, name = functools.partial(fn, omega_kind=kind), name + f"-omega{kind}"
    fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"])
    torch.cuda.synchronize()
    rt.profile_begin()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn(A, c["ranks"], c["p"], c["q"], c["omega_seed"])
    e1.record()
    torch.cuda.synchronize()
    st = rt.profile_end()
    out = {"config": name, "ms_per_solve": e0.elapsed_time(e1) / reps, "launches": st.launches}
    for k, nm in enumerate(["sketch", "power", "shrink", "small"]):
        out[nm] = [round(st.ms[k][j] / reps, 3) for j in range(len(c["dims"]))]
    print(json.dumps(out))


if __name__ == "__main__":
    main()

"""CUDA-graph replay of repeated solves (rtk_api.cu solve_entry): a key's first call runs directly,
the second captures and launches the graph, later calls replay it.  Replays must be bit-identical
to the direct path (RTK_GRAPH=0) on every algorithm and streaming engine, must read the CURRENT
contents of A (pointers are captured, not data), and keys must separate different seeds / options /
environment overrides."""
import numpy as np
import pytest

from workloads import CONFIGS, make_config_tensor
from tests.gpu_util import cuda_or_skip, to_device_colmajor

pytestmark = pytest.mark.gpu

CASES = [
    # (config recipe, dims, ranks, p, q, kwargs)
    ("c1", None, (5, 5, 5), 5, 2, dict(sequential=False)),                 # Alg. 3, concurrent mode streams
    ("c4", (40, 36, 32, 30), (6, 5, 5, 4), 4, 3, dict(sequential=True)),   # Alg. 4, d = 4, one-CTA engine
    ("c5", (300, 120, 80), (20, 10, 8), 6, 2, dict(sequential=True)),      # fp16 CTA-pair engine (mode 1)
    ("c3", (96, 80, 64), (8, 8, 8), 4, 2, dict(sequential=True, variant=1)),       # Alg. A.2
    ("c3", (96, 80, 64), (8, 8, 8), 4, 4, dict(sequential=True, pve_tol=1e-3)),    # Alg. B.1 (device stop flag)
    ("c3", (96, 80, 64), (8, 8, 8), 4, 2, dict(sequential=True, omega_kind=2)),    # Khatri-Rao sketch
    ("c3", (96, 80, 64), (8, 8, 8), 4, 2, dict(sequential=True, shift=False)),     # Alg. 2
]


def _alloc_out(torch, dims, ranks):
    from paper_2506_04840_b200 import as_column_major
    U = [torch.empty((r, n), dtype=torch.float32, device="cuda").t() for n, r in zip(dims, ranks)]
    core = as_column_major(torch.empty(ranks, dtype=torch.float32, device="cuda"))
    return core, U


def _snap(out):
    core, U = out
    return [core.cpu().numpy().copy()] + [u.cpu().numpy().copy() for u in U]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_graph_replay_bit_identical(case, monkeypatch):
    torch = cuda_or_skip()
    from paper_2506_04840_b200 import solve
    name, dims, ranks, p, q, kw = CASES[case]
    a = make_config_tensor(name, dims=dims)
    A = to_device_colmajor(a, torch)
    dims = list(A.shape)
    seed = CONFIGS[name]["omega_seed"]
    out = _alloc_out(torch, dims, ranks)
    monkeypatch.setenv("RTK_GRAPH", "0")
    solve(A, ranks, p, q, seed, out=out, **kw)
    torch.cuda.synchronize()
    ref = _snap(out)
    monkeypatch.delenv("RTK_GRAPH")
    # 1st call direct, 2nd captures + launches, 3rd and 4th replay
    for it in range(4):
        for t in out[1] + [out[0]]:
            t.fill_(float("nan"))
        solve(A, ranks, p, q, seed, out=out, **kw)
        torch.cuda.synchronize()
        got = _snap(out)
        for g, r in zip(got, ref):
            assert np.array_equal(g, r), f"call {it}: graph path differs from the direct path"


def test_graph_reads_current_data_and_keys(monkeypatch):
    torch = cuda_or_skip()
    from paper_2506_04840_b200 import solve
    a = make_config_tensor("c3", dims=(96, 80, 64))
    A = to_device_colmajor(a, torch)
    dims, ranks, p, q = list(A.shape), (8, 8, 8), 4, 2
    seed = CONFIGS["c3"]["omega_seed"]
    out = _alloc_out(torch, dims, ranks)
    for _ in range(3):   # the graph of this key now exists
        solve(A, ranks, p, q, seed, out=out)
    torch.cuda.synchronize()
    # new contents in the same buffer: the replay must see them
    A.mul_(-3.0).add_(0.25)
    solve(A, ranks, p, q, seed, out=out)
    torch.cuda.synchronize()
    got = _snap(out)
    monkeypatch.setenv("RTK_GRAPH", "0")
    solve(A, ranks, p, q, seed, out=out)
    torch.cuda.synchronize()
    ref = _snap(out)
    for g, r in zip(got, ref):
        assert np.array_equal(g, r)
    monkeypatch.delenv("RTK_GRAPH")
    # a different seed is a different key (different Omega)
    for s in (seed + 1, seed + 1, seed + 1):
        solve(A, ranks, p, q, s, out=out)
    torch.cuda.synchronize()
    got2 = _snap(out)
    monkeypatch.setenv("RTK_GRAPH", "0")
    solve(A, ranks, p, q, seed + 1, out=out)
    torch.cuda.synchronize()
    ref2 = _snap(out)
    for g, r in zip(got2, ref2):
        assert np.array_equal(g, r)
    assert not np.array_equal(ref2[1], ref[1])
    # an engine override is part of the key: FFMA tiles via RTK_PATH after the tcgen05 graph exists
    monkeypatch.delenv("RTK_GRAPH")
    monkeypatch.setenv("RTK_PATH", "ffma")
    for _ in range(3):
        solve(A, ranks, p, q, seed + 1, out=out)
    torch.cuda.synchronize()
    got3 = _snap(out)
    monkeypatch.setenv("RTK_GRAPH", "0")
    solve(A, ranks, p, q, seed + 1, out=out)
    torch.cuda.synchronize()
    ref3 = _snap(out)
    for g, r in zip(got3, ref3):
        assert np.array_equal(g, r)


def test_graph_with_report_and_side_stream():
    torch = cuda_or_skip()
    from paper_2506_04840_b200 import solve
    a = make_config_tensor("c1")
    A = to_device_colmajor(a, torch)
    c = CONFIGS["c1"]
    out = _alloc_out(torch, list(A.shape), c["ranks"])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            solve(A, c["ranks"], c["p"], c["q"], c["omega_seed"], out=out, sequential=False)
    s.synchronize()
    got = _snap(out)
    # a report call bypasses the graph (host sync) and must agree with it
    core, U, rep = solve(A, c["ranks"], c["p"], c["q"], c["omega_seed"], sequential=False, report=True)
    torch.cuda.synchronize()
    ref = [core.cpu().numpy()] + [u.cpu().numpy() for u in U]
    for g, r in zip(got, ref):
        assert np.array_equal(g, r)
    assert rep.numeric == 0

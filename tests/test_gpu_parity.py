"""End-to-end parity: CUDA path (through the C ABI) vs the float64 oracle on the same
seeded inputs and the same Omega (north_star tolerances, written here):
  |RE_gpu - RE_orc| / RE_orc <= 1e-4
  principal angle(U_k^gpu, U_k^orc) <= 1e-3 rad where gap_k > 10%
  ||U_k^T U_k - I||_F <= 1e-5
"""
import numpy as np
import pytest

from oracle import metrics, tucker
from workloads import CONFIGS, make_config_tensor, orthonormal_factor, tucker_tensor
from tests.gpu_util import cuda_or_skip, to_device_colmajor

pytestmark = pytest.mark.gpu

RE_TOL = 1e-4
ANGLE_TOL = 1e-3
ORTH_TOL = 1e-5


def run_both(a, ranks, p, q, seed, sequential, shift=True):
    torch = cuda_or_skip()
    from paper_2506_04840_b200 import solve
    A = to_device_colmajor(a, torch)
    core, U, rep = solve(A, ranks, p, q, seed, sequential=sequential, shift=shift, report=True)
    torch.cuda.synchronize()
    g_core = core.cpu().numpy()
    g_U = [u.cpu().numpy() for u in U]
    fn = tucker.rsthosvd if sequential else tucker.rthosvd
    orc = fn(a, ranks, p, q, seed, shift=shift)
    return g_core, g_U, rep, orc


def check(a, ranks, p, q, seed, sequential, gaps=None, alpha_rtol=1e-3):
    g_core, g_U, rep, orc = run_both(a, ranks, p, q, seed, sequential)
    assert rep.numeric == 0
    re_g = metrics.relative_error(a, g_core, g_U)
    re_o = metrics.relative_error(a, orc.core, orc.factors)
    assert abs(re_g - re_o) <= RE_TOL * re_o + 1e-7, (re_g, re_o)
    if gaps is None:
        gaps = metrics.mode_gaps(a, ranks, orc.factors, sequential)
    for k, u in enumerate(g_U):
        assert metrics.orthonormality(u) <= ORTH_TOL
        if gaps[k] > 0.10:
            ang = metrics.max_principal_angle(orc.factors[k], u)
            assert ang <= ANGLE_TOL, (k, ang, gaps[k])
    for k, tr in enumerate(orc.traces):
        if tr.alpha and max(tr.alpha) > 0:
            np.testing.assert_allclose(rep.alpha_trace[k], tr.alpha, rtol=alpha_rtol, atol=1e-12)
    return re_g, re_o


@pytest.mark.parametrize("path", ["ffma", "tc", "fused"])
@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4"])
def test_config_parity(cfg, path, monkeypatch):
    monkeypatch.setenv("RTK_PATH", "ffma" if path == "ffma" else "tc")
    monkeypatch.setenv("RTK_FUSED", "1" if path == "fused" else "0")
    c = CONFIGS[cfg]
    a = make_config_tensor(cfg)
    check(a, c["ranks"], c["p"], c["q"], c["omega_seed"], c["algo"] == "rsthosvd")


@pytest.mark.parametrize("seq", [False, True])
@pytest.mark.parametrize("dims,ranks,p,q", [
    ((640, 40, 36), (20, 8, 6), 6, 3),        # n_1 > 512: fused engine on a 2-CTA row split
    ((1000, 30, 20), (30, 6, 5), 10, 2),      # n_1 = 1000 (the C5 mode-1 row count), l = 40
    ((40, 30), (6, 4), 2, 2),                 # d = 2, the matrix case
    ((37, 29, 23), (4, 5, 3), 3, 2),          # odd sizes: scalar loader, ragged tiles
    ((16, 12, 10, 9), (3, 2, 4, 2), 2, 3),    # d = 4
    ((260, 18, 15), (6, 5, 4), 4, 2),         # n_1 > 256 (multi-row threads)
    ((8, 300, 7), (2, 10, 3), 3, 1),          # tall middle mode, strided view
])
def test_random_shapes(seq, dims, ranks, p, q):
    rng = np.random.default_rng(sum(dims))
    cr = tuple(min(n, r + 3) for n, r in zip(dims, ranks))
    core = rng.standard_normal(cr) * np.exp(-0.3 * np.indices(cr).sum(axis=0))
    us = [orthonormal_factor(n, r, rng) for n, r in zip(dims, cr)]
    a = tucker_tensor(core, us, noise=1e-3, rng=rng)
    check(a, ranks, p, q, 77, seq, alpha_rtol=5e-3)


@pytest.mark.parametrize("seq", [False, True])
def test_exact_recovery_gpu(seq):
    """Rank-(3,4,2) Tucker tensor, l > rank: RE at float32 rounding level, orthonormal U
    (rank-deficient sketch exercises the basis-completion path)."""
    torch = cuda_or_skip()
    from paper_2506_04840_b200 import solve
    rng = np.random.default_rng(3)
    dims, ranks = (24, 20, 16), (3, 4, 2)
    core = rng.standard_normal(ranks)
    us = [orthonormal_factor(n, r, rng) for n, r in zip(dims, ranks)]
    a = tucker_tensor(core, us)
    A = to_device_colmajor(a, torch)
    g_core, g_U, rep = solve(A, ranks, 3, 2, 5, sequential=seq, report=True)
    re = metrics.relative_error(a, g_core.cpu().numpy(), [u.cpu().numpy() for u in g_U])
    assert re < 1e-5
    for u in g_U:
        assert metrics.orthonormality(u.cpu().numpy()) <= ORTH_TOL


def test_alpha_zero_matches_algorithm_2():
    c = CONFIGS["c4"]
    a = make_config_tensor("c4", dims=(40, 36, 32, 30))
    g_core, g_U, rep, orc = run_both(a, (6, 5, 4, 3), 3, 2, 9, True, shift=False)
    assert all(x == 0.0 for t in rep.alpha_trace for x in t)
    re_g = metrics.relative_error(a, g_core, g_U)
    re_o = metrics.relative_error(a, orc.core, orc.factors)
    assert abs(re_g - re_o) <= RE_TOL * re_o


def test_deterministic_repeat():
    torch = cuda_or_skip()
    from paper_2506_04840_b200 import rsthosvd
    a = make_config_tensor("c3", dims=(120, 100, 90))
    A = to_device_colmajor(a, torch)
    c1, u1 = rsthosvd(A, (10, 9, 8), 5, 2, 1)
    c2, u2 = rsthosvd(A, (10, 9, 8), 5, 2, 1)
    assert torch.equal(c1, c2) and all(torch.equal(x, y) for x, y in zip(u1, u2))

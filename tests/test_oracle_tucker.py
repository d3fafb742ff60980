"""Pins for the float64 oracle (oracle/tucker.py, oracle/metrics.py) - CPU only.

Each test pins the oracle to something other than itself: brute-force index
loops, direct summation, closed forms from the paper (Thm 2.2 PAPER.md:131-142,
Eq. (3.2), tensor B's spectrum PAPER.md:806-815), exact
recovery (north_star), the shift invariants of PAPER.md:272-289,
and convergence to deterministic T-/ST-HOSVD (Alg. 1).
"""
import itertools

import numpy as np
import pytest

from oracle import metrics, tucker
from workloads import make_config_tensor, orthonormal_factor, tucker_tensor


def rnd(shape, seed=0):
    return np.random.default_rng(seed).standard_normal(shape)


# --------------------------------------------------------------- tensor ops
@pytest.mark.parametrize("dims", [(2, 3, 4), (3, 1, 2, 5), (4, 5)])
def test_unfold_matches_kolda_bader_index(dims):
    t = rnd(dims, 1)
    d = len(dims)
    for k in range(d):
        m = tucker.unfold(t, k)
        assert m.shape == (dims[k], int(np.prod(dims)) // dims[k])
        for idx in itertools.product(*[range(n) for n in dims]):
            j, stride = 0, 1
            for mm in range(d):
                if mm == k:
                    continue
                j += idx[mm] * stride
                stride *= dims[mm]
            assert m[idx[k], j] == t[idx]
        np.testing.assert_array_equal(tucker.fold(m, k, dims), t)


def test_mode_product_direct_summation():
    t = rnd((4, 5, 6), 2)
    b = rnd((3, 5), 3)
    out = tucker.mode_product(t, b, 1)
    ref = np.zeros((4, 3, 6))
    for i in range(4):
        for jj in range(3):
            for k in range(6):
                ref[i, jj, k] = sum(t[i, x, k] * b[jj, x] for x in range(5))
    np.testing.assert_allclose(out, ref, rtol=1e-13, atol=1e-13)


def test_mode_products_commute_and_isometry():
    t = rnd((4, 5, 6), 4)
    b, c = rnd((3, 4), 5), rnd((2, 6), 6)
    x = tucker.mode_product(tucker.mode_product(t, b, 0), c, 2)
    y = tucker.mode_product(tucker.mode_product(t, c, 2), b, 0)
    np.testing.assert_allclose(x, y, rtol=1e-13, atol=1e-13)
    q = orthonormal_factor(5, 5, np.random.default_rng(0))
    assert abs(np.linalg.norm(tucker.mode_product(t, q.T, 1)) - np.linalg.norm(t)) < 1e-12


def test_sign_pin():
    u = np.array([[0.1, -0.9, 0.5], [-0.8, 0.2, -0.5], [0.3, 0.1, 0.0]])
    v = tucker.sign_pin(u)
    np.testing.assert_array_equal(v[:, 0], -u[:, 0])   # |-0.8| largest, negative -> flip
    np.testing.assert_array_equal(v[:, 1], -u[:, 1])   # -0.9
    np.testing.assert_array_equal(v[:, 2], u[:, 2])    # tie 0.5/-0.5: lowest index (+) wins


# ------------------------------------------------------------ RE evaluator
def test_relative_error_direct_reconstruction():
    rng = np.random.default_rng(8)
    a = rng.standard_normal((6, 7, 5))
    core = rng.standard_normal((3, 4, 2))
    us = [orthonormal_factor(n, r, rng) for n, r in zip((6, 7, 5), (3, 4, 2))]
    rec = np.einsum("abc,ia,jb,kc->ijk", core, *us)
    ref = np.linalg.norm(a - rec) / np.linalg.norm(a)
    assert abs(metrics.relative_error(a, core, us) - ref) < 1e-14
    assert abs(metrics.relative_error(a, np.zeros_like(core), us) - 1.0) < 1e-15


def test_principal_angle_known_rotation():
    th = 0.3
    u = np.array([[1.0, 0], [0, 1], [0, 0]])
    v = np.array([[1.0, 0], [0, np.cos(th)], [0, np.sin(th)]])
    assert abs(metrics.max_principal_angle(u, v) - th) < 1e-14
    assert metrics.max_principal_angle(u, u @ np.array([[0.6, 0.8], [-0.8, 0.6]])) < 1e-15


def _known_sv_matrix(sig, n, m, seed):
    """n x m matrix with singular values sig (descending), random orthonormal singular vectors."""
    rng = np.random.default_rng(seed)
    k = len(sig)
    return orthonormal_factor(n, k, rng) @ np.diag(sig) @ orthonormal_factor(m, k, rng).T


@pytest.mark.parametrize("n,m", [(5, 9), (9, 5)])
def test_spectral_gap_known_singular_values(n, m):
    """gap_r = (sigma_r - sigma_{r+1}) / sigma_r on matrices with known sigma.
    Probes: an off-by-one (w[r] vs w[r-1]) gives 0.1 instead of 0.375 at r = 2; working on the
    eigenvalues lambda = sigma^2 instead of sigma gives 0.609; a wide/tall transpose slip changes
    nothing only if the implementation is right for both shapes."""
    sig = np.array([10.0, 8.0, 5.0, 4.5, 1.0])
    a = _known_sv_matrix(sig, n, m, 11)
    assert abs(metrics.spectral_gap(a, 1) - 0.2) < 1e-12
    assert abs(metrics.spectral_gap(a, 2) - 0.375) < 1e-12
    assert abs(metrics.spectral_gap(a, 3) - 0.1) < 1e-12
    # sigma_6 = 0 (rank 5): the Gram's zero eigenvalues are rounding noise ~ eps lambda_1, whose
    # square root is ~1e-7 sigma_1, so the gap is 1 to that accuracy
    assert abs(metrics.spectral_gap(a, 5) - 1.0) < 1e-6


def test_spectral_gap_rank_deficient_and_full():
    sig = np.array([3.0, 2.0])
    a = _known_sv_matrix(sig, 6, 7, 12)
    assert abs(metrics.spectral_gap(a, 2) - 1.0) < 1e-6             # sigma_3 = 0: full gap
    assert metrics.spectral_gap(np.eye(4), 4) == 1.0                 # r = n: nothing discarded


def test_mode_gaps_orthogonally_decomposable_tensor():
    """A = sum_i s_i u_i o v_i o w_i with orthonormal u, v, w: every unfolding has singular values
    s (T-HOSVD gaps in closed form).  ST with U_1 = [u_1..u_3], U_2 = [v_1, v_2]: G_(2) keeps
    s_1..s_3 and G_(3) keeps s_1, s_2, so mode 3's gap at r = 2 is 1 (sigma_3 = 0) - it would be
    0.25 if mode_gaps read A instead of the shrunk G (pins the ST recursion and its factors)."""
    rng = np.random.default_rng(13)
    s = np.array([5.0, 4.0, 3.0, 2.0, 1.0, 0.5])
    dims = (9, 8, 7)
    f = [orthonormal_factor(n, len(s), rng) for n in dims]
    a = np.einsum("i,ai,bi,ci->abc", s, *f)
    gt = metrics.mode_gaps(a, (2, 3, 4), None, sequential=False)
    np.testing.assert_allclose(gt, [(4 - 3) / 4, (3 - 2) / 3, (2 - 1) / 2], rtol=0, atol=1e-10)
    gs = metrics.mode_gaps(a, (3, 2, 2), [f[0][:, :3], f[1][:, :2], f[2][:, :2]], sequential=True)
    np.testing.assert_allclose(gs, [(3 - 2) / 3, (4 - 3) / 4, 1.0], rtol=0, atol=1e-6)


# -------------------------------------------------------------- Algorithm 1
def _tensor_b(n, v, seed):
    """Tensor B of PAPER.md:806-815 at desk scale: tendiag(v) x_k A_k."""
    rng = np.random.default_rng(seed)
    d = np.zeros((n, n, n))
    for i in range(n):
        d[i, i, i] = v[i]
    us = [orthonormal_factor(n, n, rng) for _ in range(3)]
    return np.einsum("abc,ia,jb,kc->ijk", d, *us)


def test_thosvd_tensor_b_closed_form():
    n, r = 12, 4
    v = np.exp(-np.arange(1, n + 1) / 3.0)          # 'fast decay' family
    b = _tensor_b(n, v, 3)
    for seq in (False, True):
        core, us = tucker.thosvd(b, (r, r, r), sequential=seq)
        re2 = metrics.relative_error(b, core, us) ** 2
        # sigma(B_(k)) = sorted v; the exact HOSVD of a diagonal core keeps
        # exactly the r x r x r diagonal block: RE^2 = sum_{i>r} v_i^2 / sum v_i^2
        closed = np.sum(v[r:] ** 2) / np.sum(v ** 2)
        assert abs(re2 - closed) < 1e-12
        for k in range(3):
            s = np.linalg.svd(tucker.unfold(b, k), compute_uv=False)
            np.testing.assert_allclose(s, np.sort(v)[::-1], rtol=1e-11, atol=1e-14)


def test_thosvd_theorem_2_2():
    rng = np.random.default_rng(9)
    a = rng.standard_normal((7, 8, 6)) + tucker_tensor(rng.standard_normal((3, 3, 3)),
                                                      [orthonormal_factor(n, 3, rng) for n in (7, 8, 6)],
                                                      dtype=np.float64) * 10
    ranks = (3, 4, 2)
    tails = []
    for k, r in enumerate(ranks):
        s = np.linalg.svd(tucker.unfold(a, k), compute_uv=False)
        tails.append(np.sum(s[r:] ** 2))
    for seq in (False, True):
        core, us = tucker.thosvd(a, ranks, sequential=seq)
        err2 = (metrics.relative_error(a, core, us) * np.linalg.norm(a)) ** 2
        assert err2 <= sum(tails) * (1 + 1e-12)
        if not seq:
            # per-mode equality ||A x_k (I - U U^T)||^2 = tail energy (Thm 2.2)
            for k, u in enumerate(us):
                m = tucker.unfold(a, k)
                res = np.sum((m - u @ (u.T @ m)) ** 2)
                assert abs(res - tails[k]) <= 1e-10 * tails[k]


def test_st_identity_and_orthonormality():
    """||A - A_hat||^2 = sum_k discarded energies = ||A||^2 - ||G||^2 (Eq. 3.2 structure)."""
    rng = np.random.default_rng(10)
    a = rng.standard_normal((9, 8, 7, 6))
    res = tucker.rsthosvd(a, (3, 4, 2, 3), p=2, q=2, seed=11)
    err2 = (metrics.relative_error(a, res.core, res.factors) * np.linalg.norm(a)) ** 2
    disc = metrics.st_discarded_energies(a, res.factors)
    assert abs(err2 - sum(disc)) <= 1e-12 * np.sum(a ** 2)
    assert abs(err2 - (np.sum(a ** 2) - np.sum(res.core ** 2))) <= 1e-12 * np.sum(a ** 2)
    for u in res.factors:
        assert metrics.orthonormality(u) <= 1e-12


# ------------------------------------------------------------ Algorithms 3/4
def _exact_tucker(dims, ranks, seed):
    rng = np.random.default_rng(seed)
    core = rng.standard_normal(ranks)
    us = [orthonormal_factor(n, r, rng) for n, r in zip(dims, ranks)]
    return tucker_tensor(core, us, dtype=np.float64)


@pytest.mark.parametrize("algo", ["rthosvd", "rsthosvd"])
@pytest.mark.parametrize("dims,ranks,p", [((20, 18, 16), (3, 4, 2), 3), ((12, 10, 9, 8), (2, 3, 2, 2), 2),
                                          ((30, 25), (4, 5), 4)])
def test_exact_recovery(algo, dims, ranks, p):
    a = _exact_tucker(dims, ranks, 12)
    res = getattr(tucker, algo)(a, ranks, p=p, q=1, seed=13)
    assert metrics.relative_error(a, res.core, res.factors) <= 1e-10
    for u in res.factors:
        assert metrics.orthonormality(u) <= 1e-12


@pytest.mark.parametrize("seq", [False, True])
def test_converges_to_deterministic_hosvd(seq):
    """Gapped tiny tensor, large q: randomized factors -> Alg. 1 factors."""
    rng = np.random.default_rng(14)
    dims, ranks = (16, 14, 12), (3, 3, 3)
    core = np.zeros((6, 6, 6))
    for i in range(6):
        core[i, i, i] = [10.0, 8.0, 6.0, 1.0, 0.5, 0.25][i]
    us = [orthonormal_factor(n, 6, rng) for n in dims]
    a = tucker_tensor(core, us, noise=1e-3, rng=rng, dtype=np.float64)
    det_core, det_us = tucker.thosvd(a, ranks, sequential=seq)
    fn = tucker.rsthosvd if seq else tucker.rthosvd
    res = fn(a, ranks, p=2, q=40, seed=15)
    for u_d, u_r in zip(det_us, res.factors):
        assert metrics.max_principal_angle(u_d, u_r) <= 1e-10
        np.testing.assert_allclose(u_r, u_d, atol=1e-9)          # sign pin makes them equal
    np.testing.assert_allclose(res.core, det_core, atol=1e-8)


def test_shift_closed_form_rank_l():
    """If rank(M) = l the sketch spans the dominant invariant subspace, so
    Sigma(Y_t) = lambda_i - alpha and alpha_t = lambda_l/2 for every t >= 1
    (SURVEY 8(c) alpha pin).  A dropped or sign-flipped
    alpha*Q term breaks the second step."""
    rng = np.random.default_rng(16)
    n, m, l = 20, 30, 5
    m_mat = rng.standard_normal((n, l)) @ rng.standard_normal((l, m))
    lam = np.sort(np.linalg.eigvalsh(m_mat @ m_mat.T))[::-1]
    u, tr = tucker._range_finder(m_mat, r=3, p=2, q=5, seed=17, mode1=1, shift=True)
    for a_t in tr.alpha:
        assert abs(a_t - lam[l - 1] / 2) <= 1e-10 * lam[l - 1]


def test_shift_invariants_random():
    """alpha never decreases and never exceeds lambda_l(M M^T)/2."""
    viol = 0
    for s in range(30):
        rng = np.random.default_rng(100 + s)
        n, m = int(rng.integers(8, 20)), int(rng.integers(20, 60))
        sv = np.exp(-rng.uniform(0.05, 0.6) * np.arange(n))
        mm = orthonormal_factor(n, n, rng) @ np.diag(sv) @ orthonormal_factor(m, n, rng).T
        r, p = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        lam = np.sort(np.linalg.eigvalsh(mm @ mm.T))[::-1]
        _, tr = tucker._range_finder(mm, r, p, q=6, seed=s, mode1=1, shift=True)
        al = [0.0] + tr.alpha
        assert all(b >= a for a, b in zip(al, al[1:]))
        viol += sum(a > lam[r + p - 1] / 2 * (1 + 1e-12) for a in tr.alpha)
        assert tr.alpha[-1] > 0
    assert viol == 0


def test_alpha_zero_is_algorithm_2():
    """shift=False keeps alpha at 0 (Alg. 2); it is less accurate than the shift on a
    slowly decaying spectrum at equal q (PAPER.md:289 claim, median over seeds)."""
    rng = np.random.default_rng(18)
    dims = (30, 30, 30)
    sv = 1.0 / np.arange(1, 31) ** 1.0
    core = np.zeros((30, 30, 30))
    for i in range(30):
        core[i, i, i] = sv[i]
    a = tucker_tensor(core, [orthonormal_factor(30, 30, rng) for _ in range(3)], dtype=np.float64)
    re_s, re_0 = [], []
    for s in range(9):
        r1 = tucker.rsthosvd(a, (5, 5, 5), p=2, q=1, seed=s, shift=True)
        r0 = tucker.rsthosvd(a, (5, 5, 5), p=2, q=1, seed=s, shift=False)
        assert all(x == 0.0 for t in r0.traces for x in t.alpha)
        re_s.append(metrics.relative_error(a, r1.core, r1.factors))
        re_0.append(metrics.relative_error(a, r0.core, r0.factors))
    assert np.median(re_s) <= np.median(re_0) * 1.0 + 1e-15


def test_config_c1_oracle_ballpark():
    """C1 at full size: RE equals deterministic T-HOSVD's (gaps ~98%)."""
    a = make_config_tensor("c1")
    res = tucker.rthosvd(a, (5, 5, 5), p=5, q=2, seed=1002)
    det_core, det_us = tucker.thosvd(a.astype(np.float64), (5, 5, 5), sequential=False)
    re = metrics.relative_error(a, res.core, res.factors)
    re_det = metrics.relative_error(a, det_core, det_us)
    assert abs(re - re_det) <= 1e-6 * re_det
    assert 0.02 < re < 0.08


# ------------------------------------------------------------ Alg. B.1 (PVE)
# Pins for tucker._range_finder(pve_tol=...) / rsthosvd(pve=...).
def _decaying_tensor(seed, dims=(24, 20, 18), decay=0.35):
    rng = np.random.default_rng(seed)
    core = rng.standard_normal(dims) * np.exp(-decay * np.indices(dims).sum(axis=0))
    return tucker_tensor(core, [orthonormal_factor(n, n, rng) for n in dims], dtype=np.float64)


def test_pve_tiny_tol_is_algorithm_4_at_q_max():
    """No stop (tol -> 0) runs q_max steps of Alg. 4 (B.1 line 6 loop = Alg. 4 line 6)."""
    a = _decaying_tensor(31)
    full = tucker.rsthosvd(a, (4, 3, 5), p=3, q=5, seed=9)
    pve = tucker.rsthosvd(a, (4, 3, 5), p=3, q=0, seed=9, pve=(1e-300, 5))
    for t_f, t_p in zip(full.traces, pve.traces):
        assert t_p.q == 5 and t_p.alpha == t_f.alpha
    for u_f, u_p in zip(full.factors, pve.factors):
        np.testing.assert_array_equal(u_f, u_p)
    np.testing.assert_array_equal(full.core, pve.core)


def test_pve_huge_tol_stops_after_first_step():
    """sigmahat = 0 at j = 1, so max_i sigma_i = sigma_1 <= tol sigma_{r+1} stops there with
    U_k from that step (B.1 lines 9-12) and no shift update: equals Alg. 4 with q = 1."""
    a = _decaying_tensor(32)
    one = tucker.rsthosvd(a, (4, 3, 5), p=3, q=1, seed=9)
    pve = tucker.rsthosvd(a, (4, 3, 5), p=3, q=0, seed=9, pve=(1e12, 6))
    for t in pve.traces:
        assert t.q == 1 and t.alpha == [0.0]
    for u_1, u_p in zip(one.factors, pve.factors):
        np.testing.assert_array_equal(u_1, u_p)
    np.testing.assert_array_equal(one.core, pve.core)


def test_pve_closed_form_rank_l_matrix():
    """rank(M) = l: the sketch spans range(M) exactly, so Sigma_j = lambda_i - alpha_{j-1} and
    sigma = Sigma + alpha = lambda_i(M M^T) at every step (PAPER.md:272-286 with B.1 line 9).
    Step 1 compares against sigmahat = 0: it stops iff lambda_1 <= tol lambda_{r+1} (the
    (r+1)-th value, 1-based), else step 2 sees sigma == sigmahat and stops for any tol > 0."""
    rng = np.random.default_rng(33)
    n, m, r, p = 18, 40, 3, 2
    l = r + p
    sv = np.array([9.0, 5.0, 3.0, 2.0, 1.5])
    mm = orthonormal_factor(n, l, rng) @ np.diag(sv) @ orthonormal_factor(m, l, rng).T
    lam = sv ** 2                                   # eigenvalues of M M^T, descending
    ratio = lam[0] / lam[r]                         # sigma_1 / sigma_{r+1} at step 1
    for tol, q_exp in [(1e-9, 2), (0.5 * ratio, 2), (ratio * (1 - 1e-9), 2), (ratio * (1 + 1e-9), 1)]:
        _, tr = tucker._range_finder(mm, r, p, q=0, seed=5, mode1=1, shift=True, pve_tol=(tol, 8))
        assert tr.q == q_exp, (tol, tr.q)
        np.testing.assert_allclose(tr.sigma[0][:l] + 0.0, lam, rtol=1e-12)   # alpha_0 = 0
        if q_exp == 2:
            # step 2 stops before the shift update: alpha stays lambda_l / 2 (closed form above)
            assert len(tr.alpha) == 2 and tr.alpha[0] == tr.alpha[1]
            assert abs(tr.alpha[1] - lam[l - 1] / 2) <= 1e-12 * lam[0]
            np.testing.assert_allclose(tr.sigma[1][:l] + tr.alpha[0], lam, rtol=1e-12)


def test_pve_monotone_in_tol():
    """The iterates do not depend on tol until the stop, so a larger tol never stops later."""
    for s in range(8):
        rng = np.random.default_rng(200 + s)
        n, m = int(rng.integers(12, 30)), int(rng.integers(30, 80))
        sv = np.exp(-rng.uniform(0.02, 0.3) * np.arange(n))
        mm = orthonormal_factor(n, n, rng) @ np.diag(sv) @ orthonormal_factor(m, n, rng).T
        qs = []
        for tol in [1e-8, 1e-6, 1e-4, 1e-3, 1e-2, 1e-1, 1.0, 10.0]:
            _, tr = tucker._range_finder(mm, 3, 3, q=0, seed=s, mode1=1, shift=True, pve_tol=(tol, 12))
            assert 1 <= tr.q <= 12 and len(tr.alpha) == tr.q
            qs.append(tr.q)
        assert all(b <= a for a, b in zip(qs, qs[1:])), qs


def test_pve_needs_sigma_r_plus_1():
    """B.1 compares against sigma_{r_k+1}: p = 0 leaves it undefined (rejected)."""
    with pytest.raises(ValueError):
        tucker._range_finder(np.eye(6), 2, 0, q=0, seed=1, mode1=1, shift=True, pve_tol=(0.1, 3))


def _table_b1_rows():
    import os
    rows = []
    path = os.path.join(os.path.dirname(__file__), "golden", "table_b1_tensor_b.txt")
    for line in open(path):
        if line.strip() and not line.startswith("#"):
            kind, r, tol, q1, q2, q3, re = line.split()
            rows.append((kind, int(r), float(tol), (int(q1), int(q2), int(q3)), float(re)))
    return rows


def test_table_b1_tensor_b_re_is_the_optimum():
    """Tensor B is orthogonally decomposable, so the best rank-(r,r,r)
    Tucker error is sqrt(sum_{i>r} v_i^2 / sum v_i^2); every Table B.1 row read into
    tests/golden/ prints that value to its 3 digits (the PVE runs converged)."""
    from workloads import tensor_b_spectrum
    rows = _table_b1_rows()
    assert len(rows) == 16
    for kind, r, tol, qs, re in rows:
        v = tensor_b_spectrum(600, kind)
        cf = np.sqrt(np.sum(v[r:] ** 2) / np.sum(v ** 2))
        assert float(f"{cf:.2e}") == re, (kind, r, tol, cf, re)


@pytest.mark.parametrize("kind", ["slow", "fast"])
def test_pve_tensor_b_reaches_closed_form(kind):
    """Alg. B.1 on a 60^3 tensor B: RE >= the closed-form optimum and within 1e-3 of it
    for loose and tight tol (the stop rule never ends before the leading sigmas settle)."""
    from workloads import make_tensor_b, tensor_b_spectrum
    a = make_tensor_b(60, kind, 7).astype(np.float64)
    v = tensor_b_spectrum(60, kind)
    for r in (8, 15):
        cf = np.sqrt(np.sum(v[r:] ** 2) / np.sum(v ** 2))
        for tol in (0.5, 0.01):
            res = tucker.rsthosvd(a, (r, r, r), 5, 0, 3, pve=(tol, 30))
            re = metrics.relative_error(a, res.core, res.factors)
            assert cf * (1 - 1e-12) <= re <= cf * (1 + 1e-3), (kind, r, tol, re, cf)
            assert all(2 <= t.q <= 30 for t in res.traces)


# ------------------------------------------------------------ Alg. A.2 (holistic ST-HOSVD)
def test_a2_full_width_is_deterministic_sthosvd():
    """l_k = n_k: every Q_k is square orthogonal, B = A x_k Q_k^T is a rotation of A, and
    lines 14-15 reproduce Alg. 1's ST-HOSVD of A (U_k = Q_k V_k spans A's own singular
    subspaces; both sides sign-pinned)."""
    rng = np.random.default_rng(41)
    dims, ranks = (8, 8, 8), (3, 3, 3)        # one shared p = 5 gives l_k = 8 = n_k
    a = rng.standard_normal(dims) * np.exp(-0.4 * np.indices(dims).sum(axis=0))
    det_core, det_us = tucker.thosvd(a, ranks, sequential=True)
    res = tucker.rsthosvd_a2(a, ranks, p=5, q=2, seed=3)
    for u_d, u_a in zip(det_us, res.factors):
        np.testing.assert_allclose(u_a, u_d, atol=1e-10)
    np.testing.assert_allclose(res.core, det_core, atol=1e-10)


def test_a2_core_identity_and_orthonormality():
    """core = A x_1 U_1^T ... x_d U_d^T (recomputed directly) and U_k^T U_k = I."""
    rng = np.random.default_rng(42)
    dims = (14, 12, 10, 9)
    a = rng.standard_normal(dims) * np.exp(-0.3 * np.indices(dims).sum(axis=0))
    res = tucker.rsthosvd_a2(a, (3, 4, 2, 3), p=3, q=2, seed=8)
    g = a
    for k, u in enumerate(res.factors):
        assert metrics.orthonormality(u) <= 1e-12
        g = tucker.mode_product(g, u.T, k)
    np.testing.assert_allclose(res.core, g, atol=1e-12)


@pytest.mark.parametrize("shift", [True, False])
def test_a2_exact_recovery(shift):
    """A rank-(3,2,4) Tucker tensor is recovered exactly when l_k > r_k (RE at rounding)."""
    rng = np.random.default_rng(43)
    dims, ranks = (15, 13, 11), (3, 2, 4)
    core = rng.standard_normal(ranks)
    us = [orthonormal_factor(n, r, rng) for n, r in zip(dims, ranks)]
    a = tucker_tensor(core, us, dtype=np.float64)
    res = tucker.rsthosvd_a2(a, ranks, p=2, q=1, seed=4, shift=shift)
    assert metrics.relative_error(a, res.core, res.factors) <= 1e-10


def test_a2_mode1_range_finder_is_algorithm_4s():
    """Mode 1 of A.2 factors A_(1) with the same Omega_1 as Alg. 4: identical shift trace
    and the same leading subspace (lines 3-11 = Alg. 4 lines 3-11)."""
    rng = np.random.default_rng(44)
    dims = (20, 16, 12)
    a = rng.standard_normal(dims) * np.exp(-0.25 * np.indices(dims).sum(axis=0))
    r4 = tucker.rsthosvd(a, (4, 3, 3), p=3, q=3, seed=6)
    ra = tucker.rsthosvd_a2(a, (4, 3, 3), p=3, q=3, seed=6)
    assert ra.traces[0].alpha == r4.traces[0].alpha
    assert ra.traces[0].sigma_ll == r4.traces[0].sigma_ll


@pytest.mark.parametrize("kind", ["slow", "fast"])
def test_a2_tensor_b_reaches_closed_form(kind):
    """On tensor B A.2 reaches the closed-form optimum (>= it, within 1e-3)."""
    from workloads import make_tensor_b, tensor_b_spectrum
    a = make_tensor_b(50, kind, 9).astype(np.float64)
    v = tensor_b_spectrum(50, kind)
    for r in (6, 12):
        cf = np.sqrt(np.sum(v[r:] ** 2) / np.sum(v ** 2))
        res = tucker.rsthosvd_a2(a, (r, r, r), 5, 2, 3)
        re = metrics.relative_error(a, res.core, res.factors)
        assert cf * (1 - 1e-12) <= re <= cf * (1 + 1e-3), (kind, r, re, cf)


# ------------------------------------------------------------ Appendix D sketch types
@pytest.mark.parametrize("kind", [1, 2, 3])
@pytest.mark.parametrize("algo", ["t", "st", "a2"])
def test_sketch_types_exact_recovery(kind, algo):
    """Any full-rank sketch (uniform, KR-Gaussian, KR-uniform) recovers a
    rank-r Tucker tensor exactly when l_k > r_k."""
    rng = np.random.default_rng(50 + kind)
    dims, ranks = (14, 12, 10), (3, 2, 4)
    a = tucker_tensor(rng.standard_normal(ranks), [orthonormal_factor(n, r, rng) for n, r in zip(dims, ranks)],
                      dtype=np.float64)
    fn = {"t": tucker.rthosvd, "st": tucker.rsthosvd, "a2": tucker.rsthosvd_a2}[algo]
    res = fn(a, ranks, 3, 1, 12, omega_kind=kind)
    assert metrics.relative_error(a, res.core, res.factors) <= 1e-10


@pytest.mark.parametrize("kind", [2, 3])
def test_kr_sketch_tensor_b_closed_form(kind):
    """KR sketches reach tensor B's closed-form optimum like the Gaussian one (the paper's
    Appendix D finding that the RE is comparable)."""
    from workloads import make_tensor_b, tensor_b_spectrum
    a = make_tensor_b(40, "slow", 13).astype(np.float64)
    v = tensor_b_spectrum(40, "slow")
    r = 6
    cf = np.sqrt(np.sum(v[r:] ** 2) / np.sum(v ** 2))
    res = tucker.rsthosvd(a, (r, r, r), 5, 2, 3, omega_kind=kind)
    re = metrics.relative_error(a, res.core, res.factors)
    assert cf * (1 - 1e-12) <= re <= cf * (1 + 1e-3), (re, cf)


def test_a2_rank_above_unfolding_columns():
    """Alg. A.2 with p = 0 on a matrix, r_1 = 5 > the 4 columns of the l-core's mode-1 unfolding:
    U_1 keeps r_1 orthonormal columns spanning span(Q_1) and the core identity still holds."""
    rng = np.random.default_rng(45)
    a = rng.standard_normal((34, 8)) @ rng.standard_normal((8, 60))
    res = tucker.rsthosvd_a2(a, (5, 4), 0, 1, 5)
    assert res.factors[0].shape == (34, 5)
    assert metrics.orthonormality(res.factors[0]) <= 1e-12
    q1, _ = tucker._range_finder(tucker.unfold(a, 0), 5, 0, 1, 5, 1, True, full=True)
    assert metrics.max_principal_angle(q1, res.factors[0]) <= 1e-10
    g = a
    for k, u in enumerate(res.factors):
        g = tucker.mode_product(g, u.T, k)
    np.testing.assert_allclose(res.core, g, atol=1e-10)

"""Oracle: plain float64 Tucker algorithms of Che, Wei, Wu, Yan (arXiv 2506.04840).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Slow and obviously
correct: every step follows the paper's algorithm in its own order and
notation; LAPACK (numpy.linalg.svd) is the econ-SVD primitive, like MATLAB's
``svd(.,'econ')`` in the paper's experiments.

Tensors are numpy arrays indexed T[i_1,...,i_d]; storage order is irrelevant
here.  The mode-k unfolding uses the Kolda-Bader column order (lower modes
vary fastest): column
j = sum_{m != k} i_m prod_{p<m, p != k} n_p.  Modes are 0-based in Python and
1-based in the paper / the Philox counter.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .gauss import OMEGA_GAUSS, omega, sketch


# ----------------------------------------------------------------- tensor ops
def unfold(t: np.ndarray, k: int) -> np.ndarray:
    """Mode-k unfolding A_(k) (n_k x prod_{j!=k} n_j), PAPER.md:104 (0-based k)."""
    return np.moveaxis(t, k, 0).reshape(t.shape[k], -1, order="F")


def fold(m: np.ndarray, k: int, dims) -> np.ndarray:
    """Inverse of :func:`unfold` for the same column convention."""
    dims = list(dims)
    rest = dims[:k] + dims[k + 1:]
    return np.moveaxis(m.reshape([dims[k]] + rest, order="F"), 0, k)


def mode_product(t: np.ndarray, b: np.ndarray, k: int) -> np.ndarray:
    """t x_k b : unfold_k(result) = b @ unfold_k(t)."""
    dims = list(t.shape)
    out = b @ unfold(t, k)
    dims[k] = b.shape[0]
    return fold(out, k, dims)


PIN_TIE = 1e-5


def sign_pin(u: np.ndarray) -> np.ndarray:
    """SPEC.md:232 sign convention: each column's
    largest-|entry| made positive, lowest row index on ties, where entries within
    PIN_TIE (relative) of the column's largest |entry| count as tied (C6:
    fp32 data cannot order closer magnitudes, and an unstable pick flips a column)."""
    u = np.array(u, dtype=np.float64, copy=True)
    a = np.abs(u)
    cand = a >= (1.0 - PIN_TIE) * a.max(axis=0)[None, :]
    idx = np.argmax(cand, axis=0)                  # first (lowest) qualifying row
    s = np.sign(u[idx, np.arange(u.shape[1])])
    s[s == 0] = 1.0
    return u * s[None, :]


def econ_svd(y: np.ndarray):
    """[Q, Sigma, ~] = svd(y, 'econ') with Sigma descending (LAPACK)."""
    q, s, _ = np.linalg.svd(y, full_matrices=False)
    return q, s


def leading_left_vectors(m: np.ndarray, r: int) -> np.ndarray:
    """First r left singular vectors of m (n x c), r <= n: from the economy SVD when r <= c, else
    from the full SVD (the last r - c columns then span part of the null space of m^T, any
    orthonormal completion being equally valid; Alg. 1 line "U_k = first r_k left singular
    vectors", is defined for r_k <= n_k whatever the column count)."""
    q, _, _ = np.linalg.svd(m, full_matrices=r > m.shape[1])
    return q[:, :r]


# ----------------------------------------------------------------- Algorithm 1
def thosvd(a: np.ndarray, ranks, sequential: bool):
    """Deterministic T-HOSVD / ST-HOSVD, Alg. 1.

    U_k = first r_k left singular vectors of A_(k) (T) or G_(k) (ST), then
    G = G x_k U_k^T.  Returns (core, [U_k]) with sign-pinned factors.
    """
    g = np.asarray(a, dtype=np.float64)
    a64 = g
    us = []
    for k, r in enumerate(ranks):
        m = unfold(g if sequential else a64, k)
        u = sign_pin(leading_left_vectors(m, r))
        us.append(u)
        g = mode_product(g, u.T, k)
    return g, us


# ------------------------------------------------------------- Algorithms 2-4
@dataclass
class ModeTrace:
    """Per-mode record of one randomized solve (SPEC ShiftTrace analogue)."""
    l: int
    alpha: list = field(default_factory=list)     # alpha after each power step
    sigma_ll: list = field(default_factory=list)  # Sigma_k(l_k,l_k) of each step
    sigma: list = field(default_factory=list)     # full diag(Sigma_k) of each step
    q: int = 0                                    # power steps taken


@dataclass
class Result:
    core: np.ndarray
    factors: list
    traces: list


def _range_finder(m: np.ndarray, r: int, p: int, q: int, seed: int, mode1: int,
                  shift: bool, pve_tol=None, full: bool = False, omega_kind: int = OMEGA_GAUSS,
                  dims=None):
    """Lines 3-13 of Alg. 3 / Alg. 4 for one mode.

    m      : the matrix being factored, A_(k) (Alg. 3) or G_(k) (Alg. 4), float64
    mode1  : 1-based mode index (Philox counter word, DESIGN.md RTK-GAUSS-2)
    shift  : False -> Alg. 2 (alpha fixed at 0)
    pve_tol: (tol, q_max) -> Alg. B.1 stopping rule
    full   : return the whole n x l basis Q_k of the last iterate (Alg. A.2 line 12), unpinned
    omega_kind, dims: sketch type (gauss.OMEGA_*) and the extents of the
             tensor whose mode-mode1 unfolding m is (needed by the Khatri-Rao types)
    Returns (U_k sign-pinned n x r, ModeTrace), or (Q_k n x l, ModeTrace) with full=True.
    """
    n, cols = m.shape
    l = r + p
    if pve_tol is not None and p < 1:
        raise ValueError("Alg. B.1 compares against sigma_{r+1}: needs p >= 1")
    if omega_kind == OMEGA_GAUSS:
        om = omega(seed, mode1, 0, cols, l).astype(np.float64)  # line 3: Omega_k
    else:                                                       # Appendix D types
        om = sketch(omega_kind, seed, mode1, dims, l).astype(np.float64)
    q_mat, _ = econ_svd(m @ om)                                 # line 5
    alpha = 0.0                                                 # line 5: alpha = 0
    tr = ModeTrace(l=l)
    sig_hat = np.zeros(l)
    q_steps = q if pve_tol is None else pve_tol[1]
    for _ in range(q_steps):                                    # line 6
        y = m @ (m.T @ q_mat) - alpha * q_mat                   # line 7
        q_mat, s = econ_svd(y)
        tr.q += 1
        tr.sigma.append(s.copy())
        tr.sigma_ll.append(float(s[l - 1]))
        if pve_tol is not None:                                 # B.1 lines 9-12
            sig = s + alpha
            if np.max(np.abs(sig[:r] - sig_hat[:r])) <= pve_tol[0] * sig[r]:
                tr.alpha.append(alpha)
                break
        # line 8-9: if Sigma(l,l) > alpha: alpha = (Sigma(l,l)+alpha)/2 ;
        # degenerate guard: skip when
        # Sigma(l,l) < 1e-14 Sigma(1,1) (rank(M) < l, outside PAPER.md:272's assumption)
        if shift and s[l - 1] > alpha and not (s[l - 1] < 1e-14 * s[0]):
            alpha = (s[l - 1] + alpha) / 2.0
        tr.alpha.append(alpha)
        if pve_tol is not None:
            sig_hat = sig                                       # B.1 line 15
    if full:
        return q_mat, tr
    u = sign_pin(q_mat[:, :r])                                   # line 12: Q(:,1:r_k)
    return u, tr


def rthosvd(a: np.ndarray, ranks, p: int, q: int, seed: int, shift: bool = True,
            omega_kind: int = OMEGA_GAUSS) -> Result:
    """Alg. 3, shifted randomized T-HOSVD; shift=False is Alg. 2.

    Every mode factors the ORIGINAL A_(k); the core is A x_1 U_1^T ... x_d U_d^T
    (identity PAPER.md:130).
    """
    a64 = np.asarray(a, dtype=np.float64)
    us, trs = [], []
    for k, r in enumerate(ranks):
        u, tr = _range_finder(unfold(a64, k), r, p, q, seed, k + 1, shift,
                              omega_kind=omega_kind, dims=a64.shape)
        us.append(u)
        trs.append(tr)
    g = a64
    for k, u in enumerate(us):
        g = mode_product(g, u.T, k)
    return Result(g, us, trs)


def rsthosvd(a: np.ndarray, ranks, p: int, q: int, seed: int, shift: bool = True,
             pve=None, omega_kind: int = OMEGA_GAUSS) -> Result:
    """Alg. 4, shifted randomized ST-HOSVD, order (1..d).

    shift=False is Alg. 2's ST branch; pve=(tol, q_max) is Alg. B.1 (pinned by
    tests/test_oracle_tucker.py::test_pve_*: reductions to Alg. 4 at q_max and q = 1, the
    rank-l closed form sigma = lambda_i(M M^T), monotonicity in tol).
    G starts as A; mode k factors G_(k) then G = G x_k U_k^T (line 12).
    """
    g = np.asarray(a, dtype=np.float64)
    us, trs = [], []
    for k, r in enumerate(ranks):
        u, tr = _range_finder(unfold(g, k), r, p, q, seed, k + 1, shift, pve,
                              omega_kind=omega_kind, dims=g.shape)
        us.append(u)
        trs.append(tr)
        g = mode_product(g, u.T, k)
    return Result(g, us, trs)


def rsthosvd_a2(a: np.ndarray, ranks, p: int, q: int, seed: int, shift: bool = True,
                omega_kind: int = OMEGA_GAUSS) -> Result:
    """Alg. A.2, holistic shifted randomized ST-HOSVD; shift=False is
    Alg. A.1.  Order 1..d.

    Lines 2-13: B = A; mode k runs the shifted range finder of Alg. 4 on B_(k) with
    l_k = r_k + p columns and keeps ALL l_k columns: B = B x_k Q_k^T (so mode k+1 sees
    l_1..l_k, n_{k+1}..n_d; Omega_k has l_1..l_{k-1} n_{k+1}..n_d rows, line 3).
    Line 14: deterministic ST-HOSVD of the l_1 x ... x l_d tensor B (Alg. 1, ST branch):
    V_k = first r_k left singular vectors of G_(k), G = G x_k V_k^T.
    Line 15: U_k = Q_k V_k, sign-pinned (C6); V_k's columns carry the same signs so that the
    core stays G = A x_1 U_1^T ... x_d U_d^T.  Q_k itself is sign-pinned column by column
    before line 12 (reading C18: the paper's svd leaves the signs open, and they change
    the next mode's Gaussian sketch).
    """
    b = np.asarray(a, dtype=np.float64)
    qs, trs = [], []
    for k, r in enumerate(ranks):
        q_k, tr = _range_finder(unfold(b, k), r, p, q, seed, k + 1, shift, full=True,  # lines 3-11
                                omega_kind=omega_kind, dims=b.shape)
        # the next mode's sketch B_(k+1) Omega_{k+1} sees Q_k's column signs (not only its
        # span): pin all l_k columns as C6 pins U_k (reading C18)
        q_k = sign_pin(q_k)
        qs.append(q_k)
        trs.append(tr)
        b = mode_product(b, q_k.T, k)                                                  # line 12
    g = b
    us = []
    for k, r in enumerate(ranks):                                                      # line 14
        v = leading_left_vectors(unfold(g, k), r)
        u = qs[k] @ v                                                                  # line 15
        u_p = sign_pin(u)
        sgn = np.where(np.sum(u_p * u, axis=0) < 0.0, -1.0, 1.0)
        us.append(u_p)
        g = mode_product(g, (v * sgn).T, k)
    return Result(g, us, trs)

"""Oracle-side evaluators (float64): RE, principal angles, gaps, orthonormality.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Applied identically to the
oracle's output and to the GPU's returned (core, U_k).
"""
from __future__ import annotations

import numpy as np

from .tucker import mode_product, unfold


def relative_error(a: np.ndarray, core: np.ndarray, factors) -> float:
    """RE = ||A - A_hat||_F / ||A||_F, A_hat = G x_1 U_1 ... x_d U_d.

    Evaluated explicitly in float64 (never via ||A||^2 - ||G||^2).
    The residual is accumulated slab by slab over the last mode to bound memory.
    """
    a = np.asarray(a)
    g = np.asarray(core, dtype=np.float64)
    us = [np.asarray(u, dtype=np.float64) for u in factors]
    d = a.ndim
    # B = G x_1 U_1 ... x_{d-1} U_{d-1}   (size n_1..n_{d-1} x r_d)
    b = g
    for k in range(d - 1):
        b = mode_product(b, us[k], k)
    bmat = b.reshape(-1, g.shape[-1], order="F")               # (n_1..n_{d-1}) x r_d
    num = 0.0
    den = 0.0
    ud = us[-1]
    nd = a.shape[-1]
    step = max(1, int(2 ** 26 // max(1, bmat.shape[0])))
    for s0 in range(0, nd, step):
        s1 = min(nd, s0 + step)
        slab = np.asarray(a[..., s0:s1], dtype=np.float64).reshape(-1, s1 - s0, order="F")
        rec = bmat @ ud[s0:s1, :].T
        num += float(np.sum((slab - rec) ** 2))
        den += float(np.sum(slab ** 2))
    return float(np.sqrt(num) / np.sqrt(den))


def orthonormality(u: np.ndarray) -> float:
    """||U^T U - I||_F."""
    u = np.asarray(u, dtype=np.float64)
    return float(np.linalg.norm(u.T @ u - np.eye(u.shape[1])))


def max_principal_angle(u_ref: np.ndarray, u: np.ndarray) -> float:
    """Largest principal angle between span(u_ref) and span(u):
    theta = arcsin ||(I - P_ref) u||_2 with P_ref the projector onto an
    orthonormal basis of span(u_ref) (sine form, accurate at small angles;
    SURVEY.md 8(c) C14)."""
    qr, _ = np.linalg.qr(np.asarray(u_ref, dtype=np.float64))
    qu, _ = np.linalg.qr(np.asarray(u, dtype=np.float64))
    resid = qu - qr @ (qr.T @ qu)
    s = np.linalg.norm(resid, 2)
    return float(np.arcsin(min(1.0, s)))


def spectral_gap(m: np.ndarray, r: int) -> float:
    """(sigma_r - sigma_{r+1}) / sigma_r of matrix m (float64, via eigh of m m^T)."""
    m = np.asarray(m, dtype=np.float64)
    w = np.linalg.eigvalsh(m @ m.T)[::-1]
    w = np.sqrt(np.clip(w, 0.0, None))
    if r >= len(w):
        return 1.0
    return float((w[r - 1] - w[r]) / w[r - 1]) if w[r - 1] > 0 else 0.0


def mode_gaps(a: np.ndarray, ranks, factors, sequential: bool):
    """gap_k of the matrix each mode factors in the oracle run: A_(k) (T-HOSVD) or
    the oracle's G_(k) (ST-HOSVD), SURVEY.md 8(c) C14."""
    g = np.asarray(a, dtype=np.float64)
    out = []
    for k, r in enumerate(ranks):
        m = unfold(g if sequential else np.asarray(a, dtype=np.float64), k)
        out.append(spectral_gap(m, r))
        if sequential:
            g = mode_product(g, np.asarray(factors[k], dtype=np.float64).T, k)
    return out


def st_discarded_energies(a: np.ndarray, factors) -> list:
    """ST-HOSVD per-step discarded energy ||G_{k-1} x_k (I - U_k U_k^T)||_F^2
    (the terms of Eq. (3.2))."""
    g = np.asarray(a, dtype=np.float64)
    out = []
    for k, u in enumerate(factors):
        u = np.asarray(u, dtype=np.float64)
        m = unfold(g, k)
        res = m - u @ (u.T @ m)
        out.append(float(np.sum(res ** 2)))
        g = mode_product(g, u.T, k)
    return out

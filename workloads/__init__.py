"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no unfolding, no sketch,
no power step, no SVD of an unfolding).  It only builds input tensors from a
recipe: seeded Gaussian draws, an orthonormal basis of a Gaussian matrix
(thin QR, as the paper builds its tensor B), and the
Tucker-form synthesis A = G x_1 U_1 ... x_d U_d + noise written with einsum.

Recipes follow BASELINE.json ``configs`` (SURVEY.md 8(d) "Concrete inputs"):
indices are 1-based inside the spectra, factors are qr(N(0,1)^{n x R}).Q,
inputs are generated in float64 and rounded once to float32, data seed
1000*c+1 and Omega seed 1000*c+2 for config c.  The paper's own workloads
(real datasets Yale B / COIL-100 / DC Mall; synthetic 600^3
tensors) are not in this container; these five configs
stand in for them.

Layout: the returned array is float32, indexed A[i_1,...,i_d], Fortran order
(mode-1 fastest), i.e. exactly the column-major buffer the C ABI expects.
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    "c1": dict(algo="rthosvd", dims=(64, 64, 64), ranks=(5, 5, 5), p=5, q=2,
               recipe="tucker_noise", core_ranks=(5, 5, 5), core="gauss", noise=1e-3,
               data_seed=1001, omega_seed=1002),
    "c2": dict(algo="rthosvd", dims=(200, 200, 200), ranks=(20, 20, 20), p=10, q=3,
               recipe="tucker_noise", core_ranks=(200, 200, 200), core="inv_prod",
               noise=0.0, data_seed=2001, omega_seed=2002),
    "c3": dict(algo="rsthosvd", dims=(400, 400, 400), ranks=(30, 30, 30), p=10, q=3,
               recipe="tucker_noise", core_ranks=(40, 40, 40), core="gauss", noise=1e-2,
               data_seed=3001, omega_seed=3002),
    "c4": dict(algo="rsthosvd", dims=(80, 80, 80, 80), ranks=(10, 10, 10, 10), p=5, q=4,
               recipe="tucker_noise", core_ranks=(80, 80, 80, 80), core="exp_decay",
               noise=0.0, data_seed=4001, omega_seed=4002),
    "c5": dict(algo="rsthosvd", dims=(1000, 1000, 1000), ranks=(50, 50, 50), p=10, q=5,
               recipe="tucker_noise", core_ranks=(100, 100, 100), core="inv_sqrt_prod",
               noise=1e-3, data_seed=5001, omega_seed=5002),
}


def _core(kind: str, shape, rng: np.random.Generator) -> np.ndarray:
    z = rng.standard_normal(size=shape)            # i.i.d. N(0,1)
    idx = np.meshgrid(*[np.arange(1, s + 1, dtype=np.float64) for s in shape], indexing="ij")
    if kind == "gauss":
        return z
    if kind == "inv_prod":                          # z / (i j k)
        den = np.ones(shape)
        for ix in idx:
            den = den * ix
        return z / den
    if kind == "inv_sqrt_prod":                     # z / sqrt(i j k)
        den = np.ones(shape)
        for ix in idx:
            den = den * ix
        return z / np.sqrt(den)
    if kind == "exp_decay":                         # z exp(-0.2 (i+j+k+l))
        s = np.zeros(shape)
        for ix in idx:
            s = s + ix
        return z * np.exp(-0.2 * s)
    raise ValueError(kind)


def orthonormal_factor(n: int, r: int, rng: np.random.Generator) -> np.ndarray:
    """qr(N(0,1)^{n x r}).Q  (thin QR; PAPER.md:808-810 builds tensor B this way)."""
    q, _ = np.linalg.qr(rng.standard_normal(size=(n, r)))
    return q


def tucker_tensor(core: np.ndarray, factors, noise: float = 0.0, rng=None,
                  dtype=np.float32) -> np.ndarray:
    """A = core x_1 U_1 ... x_d U_d + noise * N(0,1), float64 build, one rounding.

    Built slab by slab over the last mode so the float64 working set stays
    bounded; returns a Fortran-ordered array of ``dtype``.
    """
    d = core.ndim
    dims = tuple(u.shape[0] for u in factors)
    letters = "abcdefgh"[:d]
    # B = core x_1 U_1 ... x_{d-1} U_{d-1}   (n_1..n_{d-1} x r_d)
    b = core
    for k in range(d - 1):
        u = factors[k]
        src = letters
        dst = letters[:k] + "z" + letters[k + 1:]
        b = np.einsum(f"{src},z{letters[k]}->{dst}", b, u, optimize=True)
    out = np.empty(dims, dtype=dtype, order="F")
    nd = dims[-1]
    slab_elems = int(np.prod(dims[:-1]))
    step = max(1, (1 << 26) // max(1, slab_elems))
    ud = factors[-1]
    bmat = b.reshape(slab_elems, core.shape[-1], order="F")
    for s0 in range(0, nd, step):
        s1 = min(nd, s0 + step)
        slab = bmat @ ud[s0:s1, :].T                 # (prod n_<d) x (s1-s0)
        if noise:
            slab = slab + noise * rng.standard_normal(size=slab.shape)
        out[..., s0:s1] = slab.reshape(dims[:-1] + (s1 - s0,), order="F").astype(dtype)
    return out


def make_config_tensor(name: str, dims=None) -> np.ndarray:
    """Synthesise config ``name`` on the host (float32, Fortran order).

    ``dims`` may shrink the tensor (same recipe, core ranks clipped) for fast
    CPU tests; the default is BASELINE.json's size.
    """
    cfg = CONFIGS[name]
    dims = tuple(dims or cfg["dims"])
    rng = np.random.default_rng(cfg["data_seed"])
    cr = tuple(min(c, n) for c, n in zip(cfg["core_ranks"], dims))
    core = _core(cfg["core"], cr, rng)
    us = [orthonormal_factor(n, r, rng) for n, r in zip(dims, cr)]
    return tucker_tensor(core, us, cfg["noise"], rng)


def make_config_tensor_torch(name: str, device="cuda"):
    """Same recipe synthesised with torch on ``device`` (used for c5's 4 GB tensor,
    where a host float64 build takes minutes).  Values differ from
    :func:`make_config_tensor` (different RNG stream) but are seeded and
    deterministic; the host copy of this very tensor is what the oracle sees.
    Returns a float32 tensor of shape dims with column-major strides.
    """
    import torch
    cfg = CONFIGS[name]
    dims = tuple(cfg["dims"])
    g = torch.Generator(device=device)
    g.manual_seed(cfg["data_seed"])
    cr = tuple(min(c, n) for c, n in zip(cfg["core_ranks"], dims))
    z = torch.randn(cr, generator=g, device=device, dtype=torch.float64)
    idx = torch.meshgrid(*[torch.arange(1, s + 1, device=device, dtype=torch.float64)
                           for s in cr], indexing="ij")
    den = torch.ones(cr, device=device, dtype=torch.float64)
    for ix in idx:
        den = den * ix
    kind = cfg["core"]
    if kind == "inv_sqrt_prod":
        core = z / torch.sqrt(den)
    elif kind == "inv_prod":
        core = z / den
    elif kind == "gauss":
        core = z
    else:
        s = sum(idx)
        core = z * torch.exp(-0.2 * s)
    us = []
    for n, r in zip(dims, cr):
        q, _ = torch.linalg.qr(torch.randn((n, r), generator=g, device=device,
                                           dtype=torch.float64))
        us.append(q)
    d = len(dims)
    b = core
    letters = "abcdefgh"[:d]
    for k in range(d - 1):
        dst = letters[:k] + "z" + letters[k + 1:]
        b = torch.einsum(f"{letters},z{letters[k]}->{dst}", b, us[k])
    slab_elems = int(np.prod(dims[:-1]))
    # column-major (Fortran) buffer == C-contiguous tensor of reversed shape
    out_rev = torch.empty(tuple(reversed(dims)), device=device, dtype=torch.float32)
    bmat = b.permute(*reversed(range(d))).reshape(core.shape[-1], slab_elems)  # r_d x prod
    nd = dims[-1]
    step = max(1, (1 << 27) // slab_elems)
    for s0 in range(0, nd, step):
        s1 = min(nd, s0 + step)
        slab = us[-1][s0:s1, :] @ bmat                 # (s1-s0) x prod(n_<d), row i_d
        if cfg["noise"]:
            slab = slab + cfg["noise"] * torch.randn(slab.shape, generator=g, device=device,
                                                     dtype=torch.float64)
        out_rev.view(nd, slab_elems)[s0:s1] = slab.to(torch.float32)
    return out_rev.permute(*reversed(range(d)))        # shape dims, column-major strides


# ---------------------------------------------------------------- tensor B
def tensor_b_spectrum(n: int, kind: str) -> np.ndarray:
    """v of tensor B, i = 1..n: slow 1/i^2, fast exp(-i/7),
    sshape 0.001 + 1/(1 + exp(i - 29))."""
    i = np.arange(1, n + 1, dtype=np.float64)
    if kind == "slow":
        return 1.0 / i ** 2
    if kind == "fast":
        return np.exp(-i / 7.0)
    if kind == "sshape":
        return 0.001 + 1.0 / (1.0 + np.exp(i - 29.0))
    raise ValueError(kind)


def make_tensor_b(n: int, kind: str, seed: int, d: int = 3) -> np.ndarray:
    """B = tendiag(v, [n]*d) x_1 A_1 ... x_d A_d with A_k = orth(N(0,1)^{n x n})
    (PAPER.md:806-810); host build for small n (float32, Fortran order)."""
    rng = np.random.default_rng(seed)
    v = tensor_b_spectrum(n, kind)
    core = np.zeros((n,) * d)
    core[(np.arange(n),) * d] = v
    return tucker_tensor(core, [orthonormal_factor(n, n, rng) for _ in range(d)])


def make_tensor_b_torch(n: int, kind: str, seed: int, device="cuda"):
    """Tensor B (d = 3) built on ``device`` in float64 (the paper's 600^3 size), returned as
    a column-major float32 tensor: B = sum_i v_i a1_i o a2_i o a3_i."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    v = torch.as_tensor(tensor_b_spectrum(n, kind), device=device)
    fac = [torch.linalg.qr(torch.randn((n, n), generator=g, device=device, dtype=torch.float64))[0]
           for _ in range(3)]
    # column-major (a fastest): store as [c][b][a]
    ab = torch.einsum("ai,bi->bai", fac[0] * v, fac[1]).reshape(n * n, n)    # [(b,a)][i]
    out = (fac[2] @ ab.T).to(torch.float32)                                    # [c][(b,a)]
    return out.reshape(n, n, n).permute(2, 1, 0)

"""Oracle sketch generator: Philox4x32-10 + the frozen RTK-GAUSS-2 Box-Muller.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The paper draws "a standard Gaussian matrix Omega_k" afresh for every mode
(Alg. 3 line 3; Alg. 4 line 3; definition of a
standard Gaussian matrix PAPER.md:96).  It names no generator, so this build
freezes one (SURVEY.md 8(c) reading C2, restated in DESIGN.md "RTK-GAUSS-2"):

  key     = (lo32(seed), hi32(seed))
  counter = (c // 4, lo32(j), hi32(j), k)     j = canonical unfolding column,
                                              c = sketch column, k = 1-based mode
  x0..x3  = Philox4x32-10(counter, key)       (Salmon et al. 2011)
  (x0,x1) -> Box-Muller pair -> columns 4*(c//4)+0, +1
  (x2,x3) -> Box-Muller pair -> columns 4*(c//4)+2, +3
  u       = (2 (x >> 9) + 1) * 2^-24          (exact in binary32, u in (0,1))
  z0      = sqrt(-2 ln u_a) cos(2 pi u_b),  z1 = sqrt(-2 ln u_a) sin(2 pi u_b)

ln, sin and cos are evaluated with the fixed range reductions and fixed
polynomials below using only IEEE-754 binary32 +, -, *, / and sqrt, each
correctly rounded and never fused, in exactly the order written here; Omega_k
is the binary32 z.  The constants are the correctly rounded binary32 values of
the stated rationals, frozen as bit patterns.  The CUDA side implements the
same written spec independently (no shared code); the two must agree bit for
bit.  (RTK-GAUSS-1, the first frozen version, did the same in binary64 with
25-bit uniforms; binary32 needs about a third of the issue slots and keeps the
Gaussians accurate to a few binary32 ulp, far below what a sketch needs.)

Pins (tests/test_oracle_gauss.py): Philox against an independently compiled
cuRAND ``curand_Philox4x32_10`` and published known-answer vectors; ln/sin/cos
against libm (numpy float64) to <= 4 binary32 ulp / 3e-7; moments and a KS
test of the Gaussians.
"""
from __future__ import annotations

import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint64(0x9E3779B9)
_W1 = np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds (Salmon, Moraes, Dror, Shaw, SC'11).

    Inputs are array-likes of uint32 values (broadcast together); returns four
    uint32 arrays.  Round: (hi0,lo0)=M0*c0, (hi1,lo1)=M1*c2,
    out=(hi1^c1^k0, lo1, hi0^c3^k1, lo0); key bumped by (W0,W1) between
    rounds.
    """
    c0 = np.asarray(c0, dtype=np.uint64)
    c1 = np.asarray(c1, dtype=np.uint64)
    c2 = np.asarray(c2, dtype=np.uint64)
    c3 = np.asarray(c3, dtype=np.uint64)
    k0 = np.asarray(k0, dtype=np.uint64)
    k1 = np.asarray(k1, dtype=np.uint64)
    for rnd in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> _S32, p0 & _MASK
        hi1, lo1 = p1 >> _S32, p1 & _MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        if rnd < 9:
            k0 = (k0 + _W0) & _MASK
            k1 = (k1 + _W1) & _MASK
    return (c0.astype(np.uint32), c1.astype(np.uint32),
            c2.astype(np.uint32), c3.astype(np.uint32))


# ---- RTK-GAUSS-2 constants (binary32 bit patterns, so both sides agree) ----
def _f32(bits):
    return np.array([bits], dtype=np.uint32).view(np.float32)[0]


LN2_HI = _f32(0x3F317200)      # 0.693145751953125 (16 significant bits: n*LN2_HI exact for |n| <= 24)
LN2_LO = _f32(0x35BFBE8E)      # ln 2 - LN2_HI rounded
SQRT2 = _f32(0x3FB504F3)       # fl32(sqrt 2)
PIO2 = _f32(0x3FC90FDB)        # fl32(pi / 2)
# ln: 2 s * sum_{k=0..4} z^k/(2k+1);  sin: x * sum_{k=0..4} (-1)^k y^k/(2k+1)!;
# cos: sum_{k=0..5} (-1)^k y^k/(2k)!   (correctly rounded binary32 of each rational)
LOG_C = [_f32(b) for b in (0x3F800000, 0x3EAAAAAB, 0x3E4CCCCD, 0x3E124925, 0x3DE38E39)]
SIN_C = [_f32(b) for b in (0x3F800000, 0xBE2AAAAB, 0x3C088889, 0xB9500D01, 0x3638EF1D)]
COS_C = [_f32(b) for b in (0x3F800000, 0xBF000000, 0x3D2AAAAB, 0xBAB60B61, 0x37D00D01, 0xB493F27E)]
_F = np.float32


def _odd_int(x):
    """x (uint32) -> v = 2*(x>>9)+1, an odd integer in [1, 2^24); u = v*2^-24."""
    return (np.asarray(x, dtype=np.uint64) >> np.uint64(9)) * np.uint64(2) + np.uint64(1)


def uniform01(x):
    """u = (2(x>>9)+1)*2^-24, exact in binary32."""
    return _odd_int(x).astype(np.float32) * _F(2.0**-24)


def rtk_log_u(x):
    """ln(u) for u = (2(x>>9)+1)*2^-24 using the RTK-GAUSS-2 recipe (binary32).

    v = 2(x>>9)+1 (odd, < 2^24); e = floor(log2 v); f = v*2^-e in [1,2) (exact);
    if f > SQRT2: f = f*0.5, e = e+1 (exact);  s = (f-1)/(f+1); z = s*s;
    p = Horner(LOG_C, z); lnf = (2*s)*p;  ln u = (e-24)*LN2_HI + ((e-24)*LN2_LO + lnf).
    """
    v = _odd_int(x)
    # e = bit_length(v) - 1 = #{b in 1..23 : v >> b != 0}   (integer arithmetic)
    e = np.zeros(v.shape, dtype=np.int64)
    for b in range(1, 24):
        e += ((v >> np.uint64(b)) != 0).astype(np.int64)
    f = v.astype(np.float32) * np.ldexp(_F(1.0), -e).astype(np.float32)
    big = f > SQRT2
    f = np.where(big, f * _F(0.5), f).astype(np.float32)
    e = np.where(big, e + 1, e)
    s = (f - _F(1.0)) / (f + _F(1.0))
    z = s * s
    p = np.full_like(z, LOG_C[4])
    for k in range(3, -1, -1):
        p = p * z + LOG_C[k]
    lnf = (_F(2.0) * s) * p
    n = (e - 24).astype(np.float32)
    return n * LN2_HI + (n * LN2_LO + lnf)


def rtk_sincos_2pi_u(x):
    """(sin(2 pi u), cos(2 pi u)) for u = (2(x>>9)+1)*2^-24, RTK-GAUSS-2 recipe (binary32).

    w = 2(x>>9)+1; quadrant qd = w>>22; rem = w & (2^22-1); t = rem*2^-22 (exact);
    if rem < 2^21: x = t*PIO2, (S,C) = (sin x, cos x)
    else:          x = (1-t)*PIO2, (S,C) = (cos x, sin x)
    sin x = x*Horner(SIN_C, x*x); cos x = Horner(COS_C, x*x);
    quadrant: qd=0 -> (S,C); 1 -> (C,-S); 2 -> (-S,-C); 3 -> (-C,S)  as (sin,cos).
    """
    w = _odd_int(x)
    qd = (w >> np.uint64(22)).astype(np.int64)
    rem = w & np.uint64((1 << 22) - 1)
    t = rem.astype(np.float32) * _F(2.0**-22)
    low = rem < np.uint64(1 << 21)
    xr = np.where(low, t, _F(1.0) - t).astype(np.float32) * PIO2
    y = xr * xr
    ps = np.full_like(y, SIN_C[4])
    for k in range(3, -1, -1):
        ps = ps * y + SIN_C[k]
    sx = xr * ps
    pc = np.full_like(y, COS_C[5])
    for k in range(4, -1, -1):
        pc = pc * y + COS_C[k]
    cx = pc
    S = np.where(low, sx, cx)
    C = np.where(low, cx, sx)
    sin_o = np.select([qd == 0, qd == 1, qd == 2, qd == 3], [S, C, -S, -C]).astype(np.float32)
    cos_o = np.select([qd == 0, qd == 1, qd == 2, qd == 3], [C, -S, -C, S]).astype(np.float32)
    return sin_o, cos_o


def box_muller(xa, xb):
    """RTK-GAUSS-2 pair: r = sqrt(-2*ln u_a); (r*cos(2 pi u_b), r*sin(2 pi u_b)) in binary32."""
    r = np.sqrt(_F(-2.0) * rtk_log_u(xa))
    s, c = rtk_sincos_2pi_u(xb)
    return r * c, r * s


def omega(seed: int, mode: int, row0: int, rows: int, l: int) -> np.ndarray:
    """Rows [row0, row0+rows) of Omega_k (float32, shape rows x l).

    Row index = canonical unfolding column j (Kolda-Bader order, SURVEY.md 8(c)
    C3); mode = 1-based mode index k in processing order.  Follows PAPER.md:257
    ("Draw a standard Gaussian matrix Omega_k") with the RTK-GAUSS-2 stream.
    """
    j = np.arange(row0, row0 + rows, dtype=np.uint64)
    n4 = (l + 3) // 4
    jj = j[:, None]
    c4 = np.arange(n4, dtype=np.uint64)[None, :]
    k0 = np.uint64(seed & 0xFFFFFFFF)
    k1 = np.uint64((seed >> 32) & 0xFFFFFFFF)
    x0, x1, x2, x3 = philox4x32_10(c4, jj & _MASK, jj >> _S32, np.uint64(mode), k0, k1)
    z0, z1 = box_muller(x0, x1)
    z2, z3 = box_muller(x2, x3)
    out = np.empty((rows, n4 * 4), dtype=np.float64)
    out[:, 0::4] = z0
    out[:, 1::4] = z1
    out[:, 2::4] = z2
    out[:, 3::4] = z3
    return out[:, :l].astype(np.float32)


# ------------------------------------------------------------------ other sketch types
# PAPER.md:1377-1379 (Appendix D) compares Omega_k drawn as: a standard Gaussian matrix (the
# main algorithms, RTK-GAUSS-2 above), a uniform random matrix (entries i.i.d. U[-1, 1]), and
# the Khatri-Rao product of standard Gaussian / uniform matrices.  The paper fixes neither a
# generator nor the Khatri-Rao ordering; this build freezes (readings C2, C19):
#
# RTK-UNIF-1  counter (c // 4, lo32(j), hi32(j), 0x55000000 | k); word t of the Philox output
#             gives column 4 (c // 4) + t:  w = 2 u - 1 = (2 (x >> 8) + 1 - 2^24) 2^-24 (exact)
# RTK-KR-1    Omega_k(j, c) = fl32( prod_{m != k, m ascending} f_m(i_m, c) ), the product taken
#             in binary64, where j = sum_m i_m stride_m over the unfolding's column modes
#             (Kolda-Bader: lower modes fastest, extents of the CURRENT tensor), i.e. the
#             Khatri-Rao product F_d (.) ... (.) F_1 without F_k.  f_m is an n_m x l matrix
#             drawn row by row like Omega itself with counter word 3 =
#             0x4B000000 | (m << 8) | k  (Gaussian, RTK-GAUSS-2 pairs) or
#             0x4C000000 | (m << 8) | k  (uniform, RTK-UNIF-1 words).
OMEGA_GAUSS, OMEGA_UNIF, OMEGA_KR_GAUSS, OMEGA_KR_UNIF = 0, 1, 2, 3


def _philox_rows(seed: int, word3: int, row0: int, rows: int, l: int):
    j = np.arange(row0, row0 + rows, dtype=np.uint64)[:, None]
    c4 = np.arange((l + 3) // 4, dtype=np.uint64)[None, :]
    k0 = np.uint64(seed & 0xFFFFFFFF)
    k1 = np.uint64((seed >> 32) & 0xFFFFFFFF)
    return philox4x32_10(c4, j & _MASK, j >> _S32, np.uint64(word3), k0, k1)


def _interleave(zs, rows: int, l: int) -> np.ndarray:
    out = np.empty((rows, 4 * zs[0].shape[1]), dtype=np.float64)
    for t in range(4):
        out[:, t::4] = zs[t]
    return out[:, :l]


def unif_sym(x):
    """RTK-UNIF-1 value 2u - 1 for u = ((x>>8)+0.5) 2^-24 (exact in binary64 and binary32)."""
    return (2.0 * (np.asarray(x, dtype=np.uint64) >> np.uint64(8)).astype(np.float64) + 1.0 - 2.0 ** 24) * 2.0 ** -24


def draw_rows(seed: int, word3: int, row0: int, rows: int, l: int, uniform: bool) -> np.ndarray:
    """Rows [row0, row0+rows) x l of one Philox stream (binary64 values before rounding)."""
    x = _philox_rows(seed, word3, row0, rows, l)
    if uniform:
        return _interleave([unif_sym(v) for v in x], rows, l)
    z0, z1 = box_muller(x[0], x[1])
    z2, z3 = box_muller(x[2], x[3])
    return _interleave([z0, z1, z2, z3], rows, l)


def omega_uniform(seed: int, mode: int, row0: int, rows: int, l: int) -> np.ndarray:
    """Rows of a uniform U[-1, 1] Omega_k (RTK-UNIF-1), float32."""
    return draw_rows(seed, 0x55000000 | mode, row0, rows, l, True).astype(np.float32)


def kr_factor(seed: int, mode: int, fmode: int, n: int, l: int, uniform: bool) -> np.ndarray:
    """Factor F_m (n x l, float32) of mode k's Khatri-Rao sketch (RTK-KR-1); fmode = m (1-based)."""
    w3 = (0x4C000000 if uniform else 0x4B000000) | (fmode << 8) | mode
    return draw_rows(seed, w3, 0, n, l, uniform).astype(np.float32)


def sketch(kind: int, seed: int, mode: int, dims, l: int, row0: int = 0, rows=None) -> np.ndarray:
    """Rows [row0, row0+rows) of Omega_k (float32, rows x l) for the mode-k unfolding of a tensor
    of extents ``dims`` (d entries; mode = k, 1-based).  kind: OMEGA_* above."""
    cm = [m for m in range(1, len(dims) + 1) if m != mode]
    m_tot = int(np.prod([dims[m - 1] for m in cm]))
    rows = m_tot - row0 if rows is None else rows
    if kind == OMEGA_GAUSS:
        return omega(seed, mode, row0, rows, l)
    if kind == OMEGA_UNIF:
        return omega_uniform(seed, mode, row0, rows, l)
    uniform = kind == OMEGA_KR_UNIF
    j = np.arange(row0, row0 + rows, dtype=np.int64)
    prod = np.ones((rows, l), dtype=np.float64)
    stride = 1
    for m in cm:                                   # ascending: the fastest column mode first
        n_m = dims[m - 1]
        f = kr_factor(seed, mode, m, n_m, l, uniform).astype(np.float64)
        prod = prod * f[(j // stride) % n_m, :]
        stride *= n_m
    return prod.astype(np.float32)

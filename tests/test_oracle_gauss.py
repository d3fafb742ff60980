"""Pins for the oracle's sketch generator (oracle/gauss.py) - CPU only.

Philox4x32-10 is pinned to (a) the Random123 known-answer vectors published
with Salmon et al. (SC'11) and (b) NVIDIA cuRAND's independent implementation
compiled for the host; the RTK-GAUSS-2 (binary32) ln/sin/cos to libm; the Gaussians to
their first moments and a KS test (SPEC.md:120 moment check).
"""
import os
import shutil
import subprocess

import numpy as np
import pytest
from scipy import stats

from oracle import gauss as g

HERE = os.path.dirname(os.path.abspath(__file__))

# Random123 kat_vectors, philox4x32 R=10 (ctr, key) -> out
KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
    ((0xffffffff,) * 4, (0xffffffff, 0xffffffff), (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
    ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
     (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_known_answers(ctr, key, out):
    got = g.philox4x32_10(*ctr, *key)
    assert tuple(int(x) for x in got) == out


@pytest.fixture(scope="module")
def curand_host(tmp_path_factory):
    cxx = shutil.which("g++")
    inc = "/usr/local/cuda/include"
    if cxx is None or not os.path.exists(os.path.join(inc, "curand_philox4x32_x.h")):
        pytest.skip("no host compiler / cuRAND header")
    exe = str(tmp_path_factory.mktemp("philox") / "philox_ref")
    subprocess.check_call([cxx, "-O1", "-I", inc, os.path.join(HERE, "curand_philox_host.cpp"),
                           "-o", exe])
    return exe


def test_philox_matches_curand(curand_host):
    rng = np.random.default_rng(7)
    a = rng.integers(0, 2**32, size=(4000, 6), dtype=np.uint64)
    a[:8, :] = 0
    a[8:16, :] = 2**32 - 1
    inp = "\n".join(" ".join(str(int(v)) for v in row) for row in a) + "\n"
    out = subprocess.run([curand_host], input=inp, capture_output=True, text=True, check=True).stdout
    ref = np.array([[int(t) for t in line.split()] for line in out.strip().splitlines()],
                   dtype=np.uint64)
    got = np.stack(g.philox4x32_10(a[:, 0], a[:, 1], a[:, 2], a[:, 3], a[:, 4], a[:, 5]),
                   axis=1).astype(np.uint64)
    np.testing.assert_array_equal(got, ref)


def _all_x(step=4099):
    return np.arange(0, 2**32, step, dtype=np.uint64)


def test_uniform_exact_and_open():
    x = np.array([0, 511, 512, 2**32 - 1], dtype=np.uint64)
    u = g.uniform01(x)
    assert u.dtype == np.float32
    assert u[0] == 2.0**-24 and u[1] == 2.0**-24
    assert u[2] == 3 * 2.0**-24
    assert u[3] == 1.0 - 2.0**-24
    assert np.all((u > 0) & (u < 1))


def test_log_matches_libm():
    x = _all_x()
    u = g.uniform01(x).astype(np.float64)        # exact
    ref = np.log(u)                               # binary64 libm
    got = g.rtk_log_u(x)
    assert got.dtype == np.float32
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)   # binary32 ulp of ln u
    assert np.max(np.abs(got.astype(np.float64) - ref) / ulp) <= 4.0


def test_sincos_matches_libm():
    x = _all_x()
    u = g.uniform01(x)
    s, c = g.rtk_sincos_2pi_u(x)
    assert s.dtype == np.float32 and c.dtype == np.float32
    # reference angle from the exact odd integer, in extended precision
    th = 2.0 * np.pi * u.astype(np.longdouble)
    s, c = s.astype(np.float64), c.astype(np.float64)
    assert np.max(np.abs(s - np.sin(th).astype(np.float64))) <= 3e-7   # ~2.5 binary32 ulp at 1
    assert np.max(np.abs(c - np.cos(th).astype(np.float64))) <= 3e-7
    assert np.max(np.abs(s * s + c * c - 1.0)) <= 1e-6


def test_sincos_quadrant_special_points():
    # w = 2^22 -> u = 1/4 exactly is impossible (w odd); check the neighbours of the
    # quadrant boundaries keep the correct signs.
    for w, sgn_s, sgn_c in [((1 << 22) - 1, 1, 1), ((1 << 22) + 1, 1, -1),
                            ((1 << 23) - 1, 1, -1), ((1 << 23) + 1, -1, -1),
                            ((3 << 22) - 1, -1, -1), ((3 << 22) + 1, -1, 1)]:
        x = np.array([((w - 1) // 2) << 9], dtype=np.uint64)
        s, c = g.rtk_sincos_2pi_u(x)
        assert np.sign(s[0]) == sgn_s and np.sign(c[0]) == sgn_c


def test_gaussian_moments_and_ks():
    z = g.omega(123456789, 2, 0, 60000, 16).astype(np.float64).ravel()
    assert abs(z.mean()) < 0.01
    assert abs(z.var() - 1.0) < 0.01
    assert abs(stats.skew(z)) < 0.02
    assert abs(stats.kurtosis(z)) < 0.05
    assert stats.kstest(z, "norm").pvalue > 1e-3


def test_omega_layout_and_determinism():
    a = g.omega(42, 3, 100, 50, 15)
    b = g.omega(42, 3, 0, 200, 15)
    assert a.dtype == np.float32 and a.shape == (50, 15)
    np.testing.assert_array_equal(a, b[100:150])
    # ragged l: the first 15 columns of l=16 equal l=15
    c = g.omega(42, 3, 0, 200, 16)
    np.testing.assert_array_equal(c[:, :15], b)
    # different mode or seed -> different stream
    assert not np.array_equal(g.omega(42, 2, 0, 200, 15), b)
    assert not np.array_equal(g.omega(43, 3, 0, 200, 15), b)
    # rows past 2^32 use the hi word of the counter
    hi = g.omega(42, 1, 2**32 + 5, 3, 4)
    lo = g.omega(42, 1, 5, 3, 4)
    assert not np.array_equal(hi, lo)


def test_gaussian_tail_bound():
    """u >= 2^-24 bounds |z| by sqrt(-2 ln 2^-24) = 5.77 (the largest the spec can draw)."""
    x = np.array([0, 2**32 - 1], dtype=np.uint64)
    r = np.sqrt(-2.0 * g.rtk_log_u(x).astype(np.float64))
    assert abs(r[0] - np.sqrt(-2.0 * np.log(2.0**-24))) < 1e-5
    z = g.omega(7, 1, 0, 20000, 64)
    assert np.max(np.abs(z)) <= r[0] + 1e-5


def test_omega_golden_prefix():
    """Golden prefix written by scripts/make_golden.py from oracle/ only."""
    path = os.path.join(HERE, "golden", "omega_prefix.txt")
    rows = [l.split() for l in open(path) if l.strip() and not l.startswith("#")]
    for r in rows:
        seed, mode, j, c, hexbits = int(r[0]), int(r[1]), int(r[2]), int(r[3]), r[4]
        v = g.omega(seed, mode, j, 1, c + 1)[0, c]
        assert v.view(np.uint32) == np.uint32(int(hexbits, 16)), r


# ------------------------------------------------ Appendix D sketch types
def test_uniform_counter_layout_via_curand(curand_host):
    """RTK-UNIF-1 words come from the cuRAND Philox on counter (c//4, lo32 j, hi32 j,
    0x55000000|k) and map to (2 (x>>8) + 1 - 2^24) 2^-24 (independent Philox implementation)."""
    seed, mode, rows, l = 0x1234567890ABCDEF, 3, 7, 9
    j0 = 2**32 - 3                                   # rows straddle the hi word of the counter
    lines = []
    for j in range(j0, j0 + rows):
        for c4 in range((l + 3) // 4):
            lines.append(f"{c4} {j & 0xffffffff} {j >> 32} {0x55000000 | mode} {seed & 0xffffffff} {seed >> 32}")
    out = subprocess.run([curand_host], input="\n".join(lines) + "\n", capture_output=True, text=True,
                         check=True).stdout.split()
    words = np.array([int(t) for t in out], dtype=np.int64).reshape(rows, -1)[:, :l]
    expect = ((2 * (words >> 8) + 1 - 2**24) / 2.0**24).astype(np.float32)
    np.testing.assert_array_equal(g.omega_uniform(seed, mode, j0, rows, l), expect)


def test_uniform_moments_and_ks():
    w = g.omega_uniform(99, 2, 0, 50000, 12).astype(np.float64).ravel()
    assert w.min() > -1.0 and w.max() < 1.0
    assert abs(w.mean()) < 0.01 and abs(w.var() - 1.0 / 3.0) < 0.01
    assert stats.kstest(w, "uniform", args=(-1.0, 2.0)).pvalue > 1e-3
    assert np.all(np.mod(w * 2.0**24, 2.0) == 1.0)          # odd multiples of 2^-24


@pytest.mark.parametrize("kind", [g.OMEGA_KR_GAUSS, g.OMEGA_KR_UNIF])
def test_khatri_rao_structure(kind):
    """Every column of a KR sketch, folded to the column modes' extents, is a rank-1 tensor
    whose factors are the F_m columns (Khatri-Rao product, lower modes fastest)."""
    dims, mode, l = (6, 5, 4, 3), 2, 7
    om = g.sketch(kind, 5, mode, dims, l).astype(np.float64)
    ext = [dims[m - 1] for m in (1, 3, 4)]
    assert om.shape == (int(np.prod(ext)), l)
    uni = kind == g.OMEGA_KR_UNIF
    fs = [g.kr_factor(5, mode, m, dims[m - 1], l, uni).astype(np.float64) for m in (1, 3, 4)]
    for c in range(l):
        t = om[:, c].reshape(ext, order="F")
        outer = np.einsum("a,b,c->abc", fs[0][:, c], fs[1][:, c], fs[2][:, c])
        np.testing.assert_allclose(t, outer, rtol=1e-7, atol=0)
        sv = np.linalg.svd(t.reshape(ext[0], -1, order="F"), compute_uv=False)
        assert sv[1] <= 1e-6 * sv[0]


def test_khatri_rao_factor_distributions():
    fg = np.concatenate([g.kr_factor(11, 1, m, 4000, 8, False).ravel() for m in (2, 3)]).astype(np.float64)
    assert abs(fg.mean()) < 0.02 and abs(fg.var() - 1.0) < 0.02
    assert stats.kstest(fg, "norm").pvalue > 1e-3
    fu = g.kr_factor(11, 1, 2, 20000, 8, True).astype(np.float64).ravel()
    assert stats.kstest(fu, "uniform", args=(-1.0, 2.0)).pvalue > 1e-3
    # factor streams differ by mode pair and from the dense Omega stream
    assert not np.array_equal(g.kr_factor(11, 1, 2, 50, 8, False), g.kr_factor(11, 1, 3, 50, 8, False))
    assert not np.array_equal(g.kr_factor(11, 1, 2, 50, 8, False), g.omega(11, 1, 0, 50, 8))

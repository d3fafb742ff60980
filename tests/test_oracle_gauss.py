"""Pins for the oracle's sketch generator (oracle/gauss.py) - CPU only.

Philox4x32-10 is pinned to (a) the Random123 known-answer vectors published
with Salmon et al. (SC'11) and (b) NVIDIA cuRAND's independent implementation
compiled for the host; the RTK-GAUSS-1 ln/sin/cos to libm; the Gaussians to
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
    x = np.array([0, 255, 256, 2**32 - 1], dtype=np.uint64)
    u = g.uniform01(x)
    assert u[0] == 2.0**-25 and u[1] == 2.0**-25
    assert u[2] == 3 * 2.0**-25
    assert u[3] == 1.0 - 2.0**-25
    assert np.all((u > 0) & (u < 1))


def test_log_matches_libm():
    x = _all_x()
    u = g.uniform01(x)
    ref = np.log(u)
    got = g.rtk_log_u(x)
    ulp = np.abs(np.spacing(ref))
    assert np.max(np.abs(got - ref) / ulp) <= 4.0


def test_sincos_matches_libm():
    x = _all_x()
    u = g.uniform01(x)
    s, c = g.rtk_sincos_2pi_u(x)
    # reference angle from the exact odd integer, in extended precision
    th = 2.0 * np.pi * u.astype(np.longdouble)
    assert np.max(np.abs(s - np.sin(th).astype(np.float64))) <= 2e-15
    assert np.max(np.abs(c - np.cos(th).astype(np.float64))) <= 2e-15
    assert np.max(np.abs(s * s + c * c - 1.0)) <= 1e-15


def test_sincos_quadrant_special_points():
    # w = 2^23 -> u = 1/4 exactly is impossible (w odd); check the neighbours of the
    # quadrant boundaries keep the correct signs.
    for w, sgn_s, sgn_c in [((1 << 23) - 1, 1, 1), ((1 << 23) + 1, 1, -1),
                            ((1 << 24) - 1, 1, -1), ((1 << 24) + 1, -1, -1),
                            ((3 << 23) - 1, -1, -1), ((3 << 23) + 1, -1, 1)]:
        x = np.array([((w - 1) // 2) << 8], dtype=np.uint64)
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


def test_omega_golden_prefix():
    """Golden prefix written by scripts/make_golden.py from oracle/ only."""
    path = os.path.join(HERE, "golden", "omega_prefix.txt")
    rows = [l.split() for l in open(path) if l.strip() and not l.startswith("#")]
    for r in rows:
        seed, mode, j, c, hexbits = int(r[0]), int(r[1]), int(r[2]), int(r[3]), r[4]
        v = g.omega(seed, mode, j, 1, c + 1)[0, c]
        assert v.view(np.uint32) == np.uint32(int(hexbits, 16)), r

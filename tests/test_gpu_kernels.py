"""GPU kernels in isolation vs the oracle / fp64 brute force (through the C ABI)."""
import numpy as np
import pytest

from oracle import gauss
from workloads import CONFIGS
from tests.gpu_util import cuda_or_skip

pytestmark = pytest.mark.gpu


def test_omega_bit_exact_small():
    torch = cuda_or_skip()
    from paper_2506_04840_b200 import omega
    for seed, mode, row0, rows, l in [(1, 1, 0, 1000, 16), (1234567890123, 3, 5, 777, 15),
                                      (2**63 + 11, 8, 2**32 - 3, 9, 7), (0, 0, 0, 4, 1)]:
        g = omega(seed, mode, row0, rows, l).cpu().numpy()
        o = gauss.omega(seed, mode, row0, rows, l)
        np.testing.assert_array_equal(g.view(np.uint32), o.view(np.uint32))


@pytest.mark.parametrize("cfg", list(CONFIGS))
def test_omega_bit_exact_config_shapes(cfg):
    """Every (mode, m_k, l_k) the five configs draw: first, last and random rows."""
    torch = cuda_or_skip()
    from paper_2506_04840_b200 import omega
    c = CONFIGS[cfg]
    dims, ranks, p = c["dims"], c["ranks"], c["p"]
    rng = np.random.default_rng(0)
    for k in range(len(dims)):
        m = 1
        for j in range(len(dims)):
            if j != k:
                m *= ranks[j] if (c["algo"] == "rsthosvd" and j < k) else dims[j]
        l = ranks[k] + p
        starts = sorted(set([0, max(0, m - 512)] + list(rng.integers(0, max(1, m - 512), 4))))
        for r0 in starts:
            rows = min(512, m - r0)
            g = omega(c["omega_seed"], k + 1, int(r0), rows, l).cpu().numpy()
            o = gauss.omega(c["omega_seed"], k + 1, int(r0), rows, l)
            np.testing.assert_array_equal(g.view(np.uint32), o.view(np.uint32))


# Tolerances (relative Frobenius error of Y = M M^T Q vs float64):
#  FFMA  : fp32 products and fp32 accumulation over one CTA's columns, fp64 across CTAs:
#          ~ sqrt(K) * 2^-24 -> 2e-6 bound at these sizes (measured <= 2e-7).
#  tc    : 3xTF32 (hi*hi + hi*lo + lo*hi, the lo plane of the streamed operand itself rounded
#          to tf32: ~2^-21 per product) with the tensor core's fp32 accumulation over K = n
#          (op1) and K = m / #CTAs (op2): bound 4e-5 (measured <= 1.6e-5 at n=1000, m=2e5).
#  fused: the solver's single-pass engine (rtk_fused.cu): the same 3xTF32 products with the
#          streamed operand split in registers (exact lo) and W summed over the 2-CTA row split.
TOL = {"ffma": 2e-6, "tc": 4e-5, "fused": 4e-5}
# entry-wise, relative to the column's max |entry|: the same arithmetic, max instead of RMS
TOL_EW = {"ffma": 4e-6, "tc": 8e-5, "fused": 8e-5}


@pytest.mark.parametrize("path", ["ffma", "tc", "fused"])
@pytest.mark.parametrize("n,m,l", [(1, 7, 1), (3, 50, 2), (64, 4096, 10), (80, 1000, 15),
                                   (200, 3000, 30), (400, 2001, 40), (1000, 1234, 60),
                                   (37, 333, 13), (1500, 700, 20), (4096, 100, 8), (130, 5000, 64),
                                   (1000, 200000, 60), (256, 129, 48), (513, 777, 17), (600, 3000, 48),
                                   (1024, 4099, 33)])
def test_power_step_vs_fp64(n, m, l, path, monkeypatch):
    torch = cuda_or_skip()
    from paper_2506_04840_b200 import power_step
    monkeypatch.setenv("RTK_PATH", "ffma" if path == "ffma" else "tc")
    monkeypatch.setenv("RTK_FUSED", "1" if path == "fused" else "0")
    rng = np.random.default_rng(n * 7 + m)
    M = rng.standard_normal((n, m)).astype(np.float32)
    Q = np.linalg.qr(rng.standard_normal((n, l)))[0].astype(np.float32)
    Md = torch.from_numpy(np.asfortranarray(M)).cuda()
    Y = power_step(Md, torch.from_numpy(Q).cuda()).cpu().numpy()
    ref = M.astype(np.float64) @ (M.astype(np.float64).T @ Q.astype(np.float64))
    err = np.linalg.norm(Y - ref) / np.linalg.norm(ref)
    assert err < TOL[path], err
    # entry by entry, scaled by the column's largest |entry|: a single corrupted entry (a wrong
    # tile, a dropped K-chunk of one row) fails even where the Frobenius norm would hide it
    colmax = np.maximum(np.max(np.abs(ref), axis=0), 1e-300)
    ew = float(np.max(np.abs(Y - ref) / colmax[None, :]))
    assert ew < TOL_EW[path], ew


# The fp16 two-plane pair engine (rtk_fused2.cu, H = true): the same 22-bit split as
# 3xTF32, so the same bounds.  Forced onto the pair engine (RTK_PAIR=1) at every shape; `scale`
# multiplies M (exponent range: the power-of-two scales must follow max|M|), `spread` gives the
# columns of M magnitudes over 2^-spread .. 1 (fp16 gradual underflow of the small entries).
@pytest.mark.parametrize("n,m,l,scale,spread", [
    (3, 50, 2, 1.0, 0), (64, 4096, 10, 1.0, 0), (200, 3000, 30, 1.0, 0), (400, 2001, 40, 1.0, 0),
    (1000, 1234, 60, 1.0, 0), (37, 333, 13, 1.0, 0), (130, 5000, 64, 1.0, 0), (1000, 200000, 60, 1.0, 0),
    (256, 129, 48, 1.0, 0), (513, 777, 17, 1.0, 0), (600, 3000, 48, 1.0, 0), (1024, 4099, 33, 1.0, 0),
    (1000, 40000, 60, 1e-15, 0), (1000, 40000, 60, 1e15, 0), (700, 9000, 24, 3e-3, 20),
    (1000, 20000, 60, 1.0, 40)])
def test_power_step_f16_pair_vs_fp64(n, m, l, scale, spread, monkeypatch):
    torch = cuda_or_skip()
    from paper_2506_04840_b200 import power_step
    monkeypatch.setenv("RTK_PATH", "tc")
    monkeypatch.setenv("RTK_FUSED", "1")
    monkeypatch.setenv("RTK_PAIR", "1")
    monkeypatch.setenv("RTK_POWER_F16", "1")
    rng = np.random.default_rng(n * 11 + m)
    M = rng.standard_normal((n, m))
    if spread:
        M *= 2.0 ** (-spread * rng.random(m))[None, :]
    M = (M * scale).astype(np.float32)
    Q = np.linalg.qr(rng.standard_normal((n, l)))[0].astype(np.float32)
    Md = torch.from_numpy(np.asfortranarray(M)).cuda()
    Y = power_step(Md, torch.from_numpy(Q).cuda()).cpu().numpy()
    ref = M.astype(np.float64) @ (M.astype(np.float64).T @ Q.astype(np.float64))
    assert np.all(np.isfinite(Y))
    err = np.linalg.norm(Y - ref) / np.linalg.norm(ref)
    assert err < TOL["fused"], err
    colmax = np.maximum(np.max(np.abs(ref), axis=0), 1e-300)
    ew = float(np.max(np.abs(Y - ref) / colmax[None, :]))
    assert ew < TOL_EW["fused"], ew


# Same-sign operands (no cancellation): the tensor core's fp32 accumulator rounds toward zero, so every
# tcgen05 engine returns Y uniformly a little small, in proportion to the MMAs one accumulator receives
# (profiles/r2m_rz_probe.md: 512 x 2e5 -> 5.0e-5 on 3xTF32, 2.5e-5 on the fp16 engine, 2.9e-5 one-CTA,
# 1e-10 on the FFMA tiles).  Bounds = 2x the measured bias: a regression guard for the chain lengths, and
# the reason alpha's tolerance (rtol 1e-3) is not tightened.  The reference is the plain definition in
# float64 (numpy matmul of the same fp32 values).
@pytest.mark.parametrize("engine,env,bound", [
    ("3xTF32 pair", {"RTK_PATH": "tc", "RTK_PAIR": "1"}, 1.0e-4),
    ("fp16 pair", {"RTK_PATH": "tc", "RTK_PAIR": "1", "RTK_POWER_F16": "1"}, 5.0e-5),
    ("one-CTA fused", {"RTK_PATH": "tc", "RTK_PAIR": "0"}, 6.0e-5),
    ("FFMA tiles", {"RTK_PATH": "ffma"}, 2.0e-6),
])
def test_power_step_same_sign_bias(engine, env, bound, monkeypatch):
    torch = cuda_or_skip()
    from paper_2506_04840_b200 import power_step
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    n, m, l = 512, 200000, 60
    rng = np.random.default_rng(512)
    M = np.abs(rng.standard_normal((n, m))).astype(np.float32)
    Q = (np.abs(rng.standard_normal((n, l))) / np.sqrt(n)).astype(np.float32)
    Md = torch.from_numpy(np.asfortranarray(M)).cuda()
    Y = power_step(Md, torch.from_numpy(Q).cuda()).cpu().numpy()
    ref = M.astype(np.float64) @ (M.astype(np.float64).T @ Q.astype(np.float64))
    rel = (Y - ref) / ref
    print(f"{engine}: mean {rel.mean():+.3e} max |rel| {np.abs(rel).max():.3e}")
    assert float(np.abs(rel).max()) < bound, (engine, float(rel.mean()), float(np.abs(rel).max()))
    if "ffma" not in env.get("RTK_PATH", ""):
        assert rel.mean() < 0 and np.abs(rel).max() < 1.5 * abs(rel.mean())    # a uniform shrink, not noise


def test_power_step_padded_leading_dimension():
    torch = cuda_or_skip()
    from paper_2506_04840_b200 import power_step
    rng = np.random.default_rng(5)
    n, m, l, ld = 102, 999, 12, 104
    buf = np.zeros((ld, m), dtype=np.float32, order="F")
    buf[:n] = rng.standard_normal((n, m))
    Q = rng.standard_normal((n, l)).astype(np.float32)
    Md = torch.from_numpy(buf).cuda()[:n]
    Y = power_step(Md, torch.from_numpy(Q).cuda()).cpu().numpy()
    M = buf[:n].astype(np.float64)
    ref = M @ (M.T @ Q.astype(np.float64))
    assert np.linalg.norm(Y - ref) / np.linalg.norm(ref) < 2e-6


# ------------------------------------------------ Appendix D sketch types
@pytest.mark.parametrize("kind", [1, 2, 3])
@pytest.mark.parametrize("dims,mode,l,row0,rows", [
    ((30, 20, 10), 1, 13, 0, None),
    ((30, 20, 10), 2, 16, 7, 101),
    ((9, 8, 7, 6), 3, 21, 0, None),
    ((5, 4), 2, 3, 1, 3),
])
def test_sketch_types_bit_exact(kind, dims, mode, l, row0, rows):
    """The CUDA RTK-UNIF-1 / RTK-KR-1 generators equal the oracle's bit for bit."""
    torch = cuda_or_skip()
    from oracle import gauss
    from paper_2506_04840_b200 import sketch
    got = sketch(kind, 0xABCDEF0123, mode, dims, l, row0, rows).cpu().numpy()
    ref = gauss.sketch(kind, 0xABCDEF0123, mode, dims, l, row0, rows)
    np.testing.assert_array_equal(got.view(np.uint32), ref.view(np.uint32))

"""Multi-GPU last-mode shard of Alg. 4 (rtk_rsthosvd_shard in include/rtucker.h).

CPU (-m "not gpu"): the host-side facts the shard rests on, with real world_size-2 gloo
collectives: the slab bounds tile mode d; a last-mode slab's mode-k unfolding (k < d) is a
contiguous column range of the full unfolding, also after ST shrinks; Omega_k's rows for that range
are rows [j0, j0 + m) of the full Omega_k; and Alg. 4 run with every M (M^T Q) / M Omega formed
per slab and summed by an all-reduce equals the oracle's Alg. 4 on the whole tensor.

GPU (-m gpu): two processes on the one visible GPU, gloo all-reduce (host-staged; the kernels of
one rank never wait on the other's), each solving its slab with rtk_rsthosvd_shard; the result must
match the single-GPU solve of the whole tensor to fp32 rounding (the all-reduce changes only the
summation order of Y).
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import tucker  # noqa: E402
from oracle.gauss import omega, sketch  # noqa: E402
from paper_2506_04840_b200._lib import shard_bounds  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("n,world", [(7, 1), (7, 2), (10, 3), (1000, 8), (37, 5)])
def test_shard_bounds_tile_the_mode(n, world):
    got = [shard_bounds(n, world, r) for r in range(world)]
    assert got[0][0] == 0 and sum(c for _, c in got) == n
    for (b0, c0), (b1, _) in zip(got, got[1:]):
        assert b1 == b0 + c0
    assert max(c for _, c in got) - min(c for _, c in got) <= 1
    with pytest.raises(ValueError):
        shard_bounds(n, world, world)


def test_slab_unfolding_is_a_column_range():
    """For k < d-1, unfold(slab, k) = unfold(full, k)[:, P b : P (b + c)], P = prod_{m != k, m < d-1}
    n_m (i_d is the slowest unfolding column index) -- also for the ST-shrunk tensors."""
    rng = np.random.default_rng(3)
    dims = (5, 4, 6, 7)
    a = rng.standard_normal(dims)
    shrink = [rng.standard_normal((2, 5)), rng.standard_normal((3, 4)), rng.standard_normal((2, 6))]
    for b, c in [(0, 3), (3, 4), (2, 1)]:
        g, gs = a, a[..., b:b + c]
        for k in range(len(dims) - 1):
            p = int(np.prod([g.shape[m] for m in range(len(dims) - 1) if m != k]))
            np.testing.assert_array_equal(tucker.unfold(gs, k), tucker.unfold(g, k)[:, p * b:p * (b + c)])
            g = tucker.mode_product(g, shrink[k], k)
            gs = tucker.mode_product(gs, shrink[k], k)
        # after the last shrink: the slab is rows [b, b + c) of the mode-d unfolding
        np.testing.assert_allclose(tucker.unfold(gs, 3), tucker.unfold(g, 3)[b:b + c], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("kind", [0, 1, 2, 3])
def test_omega_rows_of_a_column_range(kind):
    dims, mode, l = (6, 5, 7), 2, 4
    full = sketch(kind, 11, mode, dims, l) if kind else omega(11, mode, 0, 42, l)
    for j0, m in [(0, 10), (12, 18), (35, 7)]:
        part = sketch(kind, 11, mode, dims, l, row0=j0, rows=m) if kind else omega(11, mode, j0, m, l)
        np.testing.assert_array_equal(part, full[j0:j0 + m])


def _sharded_rsthosvd(a_slab, full_dims, begin, ranks, p, q, seed, allreduce):
    """Alg. 4 with every product of the unfolding formed on this rank's slab and
    summed by `allreduce`, in the oracle's operations otherwise (econ SVD of each iterate, the same
    alpha rule); mode d on the all-reduced (gathered) mode-d unfolding, redundantly."""
    d = len(full_dims)
    g = np.asarray(a_slab, dtype=np.float64)
    us = []
    for k in range(d - 1):
        mk = tucker.unfold(g, k)
        l = ranks[k] + p
        stride = int(np.prod([g.shape[m] for m in range(d - 1) if m != k]))
        om = omega(seed, k + 1, stride * begin, mk.shape[1], l).astype(np.float64)
        qm, _ = tucker.econ_svd(allreduce(mk @ om))
        alpha = 0.0
        for _ in range(q):
            y = allreduce(mk @ (mk.T @ qm))
            y = y - alpha * qm
            qm, s = tucker.econ_svd(y)
            if s[l - 1] > alpha and not (s[l - 1] < 1e-14 * s[0]):
                alpha = (s[l - 1] + alpha) / 2.0
        u = tucker.sign_pin(qm[:, :ranks[k]])
        us.append(u)
        g = tucker.mode_product(g, u.T, k)
    # gather mode d: the slab's rows at [begin, begin + c), zero elsewhere, summed
    md = tucker.unfold(g, d - 1)
    full = np.zeros((full_dims[-1], md.shape[1]))
    full[begin:begin + md.shape[0]] = md
    full = allreduce(full)
    gd = tucker.fold(full, d - 1, list(g.shape[:-1]) + [full_dims[-1]])
    u, _ = tucker._range_finder(tucker.unfold(gd, d - 1), ranks[-1], p, q, seed, d, True, dims=gd.shape)
    us.append(u)
    return tucker.mode_product(gd, u.T, d - 1), us


def _gloo_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(77)
    dims, ranks = (9, 8, 10), (3, 3, 2)
    cr = (4, 4, 3)
    core = rng.standard_normal(cr)
    fac = [np.linalg.qr(rng.standard_normal((n, r)))[0] for n, r in zip(dims, cr)]
    a = tucker.mode_product(tucker.mode_product(tucker.mode_product(core, fac[0], 0), fac[1], 1), fac[2], 2)
    a = a + 1e-3 * rng.standard_normal(dims)
    b, c = shard_bounds(dims[-1], world, rank)

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x))
        dist.all_reduce(t)
        return t.numpy()

    g_core, g_us = _sharded_rsthosvd(a[..., b:b + c], dims, b, ranks, 2, 2, 5, allreduce)
    ref = tucker.rsthosvd(a, ranks, 2, 2, 5)
    out[rank] = (float(np.abs(g_core - ref.core).max() / np.abs(ref.core).max()),
                 max(float(np.abs(u - v).max()) for u, v in zip(g_us, ref.factors)))
    dist.destroy_process_group()


def test_sharded_alg4_gloo_world_size_2_equals_oracle():
    pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    for r in range(2):
        dcore, du = out[r]
        assert dcore < 1e-10 and du < 1e-10, (r, dcore, du)


# ---------------------------------------------------------------------------------------- GPU
def _gpu_worker(rank, world, port, dims, ranks, p, q, out, kind=0):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import paper_2506_04840_b200 as rt
    from tests.gpu_util import to_device_colmajor
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    rng = np.random.default_rng(sum(dims))
    cr = tuple(min(n, r + 4) for n, r in zip(dims, ranks))
    core = rng.standard_normal(cr) * np.exp(-0.2 * np.indices(cr).sum(axis=0))
    a = core
    for k, (n, r) in enumerate(zip(dims, cr)):
        a = tucker.mode_product(a, np.linalg.qr(rng.standard_normal((n, r)))[0], k)
    a = (a + 1e-3 * rng.standard_normal(dims)).astype(np.float32)
    b, c = rt.shard_bounds(dims[-1], world, rank)
    A = to_device_colmajor(a, torch)
    S = to_device_colmajor(np.ascontiguousarray(a[..., b:b + c]), torch)
    core1, u1 = rt.rsthosvd(A, ranks, p, q, 19, omega_kind=kind)
    core_s, u_s = rt.rsthosvd_shard(S, dims, b, ranks, p, q, 19, omega_kind=kind)
    torch.cuda.synchronize()
    c0, cs = core1.double().cpu().numpy(), core_s.double().cpu().numpy()
    out[rank] = (float(np.abs(cs - c0).max() / np.abs(c0).max()),
                 max(float((x - y).abs().max()) for x, y in zip(u_s, u1)),
                 float(core_s.double().norm()), float(core1.double().norm()))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("dims,ranks,p,q", [
    ((1000, 64, 40), (50, 10, 8), 10, 3),    # mode 1 on the one-CTA engine (5 pair-blocks per slab), l = 60
    ((1000, 200, 100), (30, 10, 8), 6, 2),   # mode 1 on the fp16 pair engine (39 pair-blocks per slab)
    ((120, 90, 33), (12, 9, 6), 5, 2),       # one-CTA engine, odd slab extents (17 + 16)
    ((40, 30, 20, 18), (6, 5, 4, 3), 4, 2),  # d = 4
])
def test_shard_matches_single_gpu(dims, ranks, p, q):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, dims, ranks, p, q, out)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(600)
        assert pr.exitcode == 0
    assert out[0][2] == out[1][2]            # identical outputs on both ranks
    for r in range(2):
        dcore, du, _, _ = out[r]
        assert dcore <= 2e-5 and du <= 2e-4, (r, dcore, du)


@pytest.mark.gpu
@pytest.mark.parametrize("world,kind", [(3, 0), (2, 2), (2, 1)])
def test_shard_world3_and_sketch_types(world, kind):
    """Three ranks (slabs 7 / 7 / 6 of n_3 = 20) with the Gaussian sketch, and two ranks with the
    Khatri-Rao Gaussian and the uniform sketch (Omega_k's rows for the slab's column range, with the
    Khatri-Rao factor of mode d drawn over its full extent)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    dims, ranks, p, q = (300, 40, 20), (20, 8, 5), 6, 2
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, dims, ranks, p, q, out, kind))
             for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(600)
        assert pr.exitcode == 0
    for r in range(world):
        assert out[r][2] == out[0][2]
        dcore, du, _, _ = out[r]
        assert dcore <= 2e-5 and du <= 2e-4, (r, dcore, du)

"""ctypes binding of include/rtucker.h (argument marshalling only)."""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

ABI_FUNCTIONS = ["rtk_rthosvd", "rtk_rsthosvd", "rtk_solve", "rtk_workspace_bytes", "rtk_workspace_bytes_ex",
                 "rtk_omega", "rtk_sketch", "rtk_rsthosvd_shard", "rtk_workspace_bytes_shard",
                 "rtk_power_step", "rtk_profile_begin", "rtk_profile_end", "rtk_debug_step_clocks",
                 "rtk_last_error", "rtk_version"]

RTK_STATUS = {0: "RTK_OK", 1: "RTK_ERR_ARG", 2: "RTK_ERR_SHAPE", 3: "RTK_ERR_ALIGN",
              4: "RTK_ERR_WORKSPACE", 5: "RTK_ERR_CUDA", 6: "RTK_ERR_NUMERIC"}


class RtkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{RTK_STATUS.get(code, code)}: {msg}")
        self.code = code


class _Report(ctypes.Structure):
    _fields_ = [("alpha_trace", ctypes.POINTER(ctypes.c_double)),
                ("sigma", ctypes.POINTER(ctypes.c_double)),
                ("q_used", ctypes.POINTER(ctypes.c_int32)),
                ("fallback", ctypes.c_int32),
                ("numeric", ctypes.c_int32)]


class ProfStats(ctypes.Structure):
    _fields_ = [("ms", (ctypes.c_double * 8) * 4), ("count", (ctypes.c_int32 * 8) * 4),
                ("launches", ctypes.c_int64)]


class _Options(ctypes.Structure):
    _fields_ = [("sequential", ctypes.c_int32), ("shift", ctypes.c_int32),
                ("pve_tol", ctypes.c_double), ("path", ctypes.c_int32), ("variant", ctypes.c_int32),
                ("omega", ctypes.c_int32)]


# rtk_allreduce_fn: int (*)(void* buf, int64_t count, int32_t dtype, void* stream, void* ctx)
_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p,
                                 ctypes.c_void_p)


def lib_path() -> str:
    return os.environ.get("RTUCKER_LIB", os.path.join(HERE, "librtucker.so"))


def load_library():
    """Load librtucker.so (raises loudly if it is missing: there is no fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise ImportError(f"rtucker CUDA library not built: {path} "
                          "(run `python -m paper_2506_04840_b200.build`)")
    lib = ctypes.CDLL(path)
    i64p = ctypes.POINTER(ctypes.c_int64)
    i32p = ctypes.POINTER(ctypes.c_int32)
    vp = ctypes.c_void_p
    solver_args = [vp, i64p, ctypes.c_int32, i32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64,
                   ctypes.POINTER(ctypes.c_void_p), vp, vp, ctypes.c_size_t, vp,
                   ctypes.POINTER(_Report)]
    lib.rtk_rthosvd.argtypes = solver_args
    lib.rtk_rsthosvd.argtypes = solver_args
    lib.rtk_solve.argtypes = [ctypes.POINTER(_Options)] + solver_args
    for f in (lib.rtk_rthosvd, lib.rtk_rsthosvd, lib.rtk_solve):
        f.restype = ctypes.c_int
    lib.rtk_workspace_bytes.argtypes = [ctypes.c_int32, i64p, ctypes.c_int32, i32p, ctypes.c_int32,
                                        ctypes.c_int32]
    lib.rtk_workspace_bytes.restype = ctypes.c_size_t
    lib.rtk_workspace_bytes_ex.argtypes = [ctypes.POINTER(_Options), i64p, ctypes.c_int32, i32p, ctypes.c_int32,
                                           ctypes.c_int32]
    lib.rtk_workspace_bytes_ex.restype = ctypes.c_size_t
    lib.rtk_sketch.argtypes = [ctypes.c_int32, ctypes.c_uint64, ctypes.c_int32, i64p, ctypes.c_int32,
                               ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
    lib.rtk_sketch.restype = ctypes.c_int
    lib.rtk_rsthosvd_shard.argtypes = [ctypes.POINTER(_Options), vp, i64p, ctypes.c_int32, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_int32, i32p, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p), vp, vp, ctypes.c_size_t,
                                       vp, _ALLREDUCE_FN, vp]
    lib.rtk_rsthosvd_shard.restype = ctypes.c_int
    lib.rtk_workspace_bytes_shard.argtypes = [ctypes.POINTER(_Options), i64p, ctypes.c_int32, ctypes.c_int64, i32p,
                                              ctypes.c_int32, ctypes.c_int32]
    lib.rtk_workspace_bytes_shard.restype = ctypes.c_size_t
    lib.rtk_omega.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                              ctypes.c_int32, vp, vp]
    lib.rtk_omega.restype = ctypes.c_int
    lib.rtk_power_step.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, vp,
                                   ctypes.c_int32, vp, vp]
    lib.rtk_power_step.restype = ctypes.c_int
    lib.rtk_profile_begin.argtypes = []
    lib.rtk_profile_begin.restype = ctypes.c_int
    lib.rtk_profile_end.argtypes = [ctypes.POINTER(ProfStats)]
    lib.rtk_profile_end.restype = ctypes.c_int
    lib.rtk_debug_step_clocks.argtypes = [vp]
    lib.rtk_debug_step_clocks.restype = ctypes.c_int
    lib.rtk_last_error.restype = ctypes.c_char_p
    lib.rtk_version.restype = ctypes.c_char_p
    _LIB = lib
    return lib


def profile_begin():
    """Start recording CUDA events around the library's launches (see rtk_profile_begin)."""
    _check(load_library().rtk_profile_begin())


def profile_end() -> ProfStats:
    """Stop recording; returns summed device ms / counts by (kind, mode) and #launches."""
    st = ProfStats()
    _check(load_library().rtk_profile_end(ctypes.byref(st)))
    return st


def version() -> str:
    return load_library().rtk_version().decode()


def _check(code: int):
    if code != 0:
        msg = load_library().rtk_last_error().decode()
        raise RtkError(code, msg)


def _stream_handle(device):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def as_column_major(x):
    """Return x (shape n_1..n_d) with column-major strides (mode-1 fastest), copying if needed."""
    import torch
    d = x.dim()
    rev = list(range(d - 1, -1, -1))
    return x.permute(*rev).contiguous().permute(*rev)


def _is_column_major(x) -> bool:
    s = 1
    for k in range(x.dim()):
        if x.shape[k] != 1 and x.stride(k) != s:
            return False
        s *= x.shape[k]
    return True


def workspace_bytes(sequential: bool, dims, ranks, p: int, q: int, variant: int = 0, omega_kind: int = 0,
                    path: int = 0) -> int:
    lib = load_library()
    d = len(dims)
    dd = (ctypes.c_int64 * d)(*dims)
    rr = (ctypes.c_int32 * d)(*ranks)
    opt = _Options(1 if sequential else 0, 1, 0.0, int(path), int(variant), int(omega_kind))
    n = lib.rtk_workspace_bytes_ex(ctypes.byref(opt), dd, d, rr, p, q)
    if n == 0:
        raise RtkError(1, lib.rtk_last_error().decode())
    return int(n)


def _check_outputs(core, U, dims, ranks, dev):
    """out=(core, U) are written by the kernels through raw pointers: each U[k] must be an
    n_k x r_k float32 column-major (stride(0) == 1, stride(1) == n_k) tensor on A's device, core
    an r_1 x ... x r_d float32 column-major tensor on A's device (the ABI writes U[k] with leading
    dimension n_k, so stride(1) must equal n_k)."""
    import torch
    if len(U) != len(dims):
        raise ValueError("out: need one factor per mode")
    for k, (u, n, r) in enumerate(zip(U, dims, ranks)):
        if not isinstance(u, torch.Tensor) or u.dtype != torch.float32 or u.device != dev:
            raise ValueError(f"out: U[{k}] must be a float32 tensor on {dev}")
        if tuple(u.shape) != (n, r):
            raise ValueError(f"out: U[{k}] has shape {tuple(u.shape)}, expected {(n, r)}")
        if (n > 1 and u.stride(0) != 1) or (r > 1 and u.stride(1) != n):
            raise ValueError(f"out: U[{k}] must be column-major with leading dimension n_k "
                             "(stride(0) == 1, stride(1) == n_k)")
    if not isinstance(core, torch.Tensor) or core.dtype != torch.float32 or core.device != dev:
        raise ValueError(f"out: core must be a float32 tensor on {dev}")
    if tuple(core.shape) != tuple(ranks):
        raise ValueError(f"out: core has shape {tuple(core.shape)}, expected {tuple(ranks)}")
    if not _is_column_major(core):
        raise ValueError("out: core must be column-major (use as_column_major)")


@dataclass
class Report:
    alpha_trace: list      # d lists of q alphas
    sigma: list            # d lists of l final sigma estimates (diag(Sigma)+alpha)
    q_used: list
    fallback: int
    numeric: int


class _WorkspaceCache:
    """Keeps one device workspace per (device, size) so repeated solves do not reallocate."""

    def __init__(self):
        self.buf = {}

    def get(self, device, nbytes):
        import torch
        key = str(device)
        b = self.buf.get(key)
        if b is None or b.numel() < nbytes:
            b = torch.empty(nbytes, dtype=torch.uint8, device=device)
            self.buf[key] = b
        return b


_WS = _WorkspaceCache()


def solve(A, ranks, p: int, q: int, seed: int, sequential: bool = True, shift: bool = True,
          report: bool = False, out=None, workspace=None, pve_tol: float = 0.0, path: int = 0,
          variant: int = 0, omega_kind: int = 0):
    """General solver: Alg. 4 (sequential) / Alg. 3 (not sequential); shift=False is Alg. 2.

    pve_tol > 0 selects Alg. B.1 with q as q_max (sequential only);
    path: 0 auto, 1 FP32 FFMA tiles, 2 tcgen05 3xTF32 (rtk_options.path).
    variant=1 selects Alg. A.2 (shift=False gives Alg. A.1).
    omega_kind: 0 Gaussian, 1 uniform, 2 KR-Gaussian, 3 KR-uniform sketch.

    Returns (core, [U_1..U_d]) or (core, U, Report) with report=True.
    ``out=(core, [U_k])`` reuses caller-allocated outputs (column-major).
    """
    import torch
    lib = load_library()
    if not isinstance(A, torch.Tensor) or not A.is_cuda:
        raise ValueError("A must be a CUDA torch.Tensor (no CPU fallback)")
    if A.dtype != torch.float32:
        raise ValueError("A must be float32")
    if not _is_column_major(A):
        raise ValueError("A must be column-major (mode-1 fastest); use as_column_major(A)")
    dims = [int(s) for s in A.shape]
    d = len(dims)
    ranks = [int(r) for r in ranks]
    if len(ranks) != d:
        raise ValueError("len(ranks) must equal A.dim()")
    dev = A.device
    if out is None:
        U = [torch.empty((r, n), dtype=torch.float32, device=dev).t() for n, r in zip(dims, ranks)]
        core = as_column_major(torch.empty(ranks, dtype=torch.float32, device=dev))
    else:
        core, U = out
        _check_outputs(core, U, dims, ranks, dev)
    dd = (ctypes.c_int64 * d)(*dims)
    rr = (ctypes.c_int32 * d)(*ranks)
    up = (ctypes.c_void_p * d)(*[u.data_ptr() for u in U])
    ws_bytes = workspace_bytes(sequential, dims, ranks, p, q, variant, omega_kind, path) if min(ranks) >= 1 else 0
    if workspace is not None:
        if not workspace.is_cuda or workspace.device != dev or not workspace.is_contiguous():
            raise ValueError("workspace must be a contiguous CUDA tensor on A's device")
        if workspace.numel() * workspace.element_size() < ws_bytes:
            raise ValueError(f"workspace too small: need {ws_bytes} bytes")
    ws = workspace if workspace is not None else _WS.get(dev, max(ws_bytes, 1))
    opt = _Options(1 if sequential else 0, 1 if shift else 0, float(pve_tol), int(path), int(variant),
                   int(omega_kind))
    rep = None
    bufs = None
    if report:
        at = (ctypes.c_double * (d * q))()
        sg = (ctypes.c_double * (d * 128))()
        qu = (ctypes.c_int32 * d)()
        rep = _Report(ctypes.cast(at, ctypes.POINTER(ctypes.c_double)),
                      ctypes.cast(sg, ctypes.POINTER(ctypes.c_double)),
                      ctypes.cast(qu, ctypes.POINTER(ctypes.c_int32)), 0, 0)
        bufs = (at, sg, qu)
    with torch.cuda.device(dev):
        code = lib.rtk_solve(ctypes.byref(opt), ctypes.c_void_p(A.data_ptr()), dd, d, rr, p, q,
                             ctypes.c_uint64(seed), up, ctypes.c_void_p(core.data_ptr()),
                             ctypes.c_void_p(ws.data_ptr()), ws.numel() * ws.element_size(), _stream_handle(dev),
                             ctypes.byref(rep) if rep is not None else None)
    _check(code)
    if not report:
        return core, U
    at, sg, qu = bufs
    ls = [r + p for r in ranks]
    r_obj = Report([list(at[k * q:(k + 1) * q]) for k in range(d)],
                   [list(sg[k * 128:k * 128 + ls[k]]) for k in range(d)],
                   list(qu), rep.fallback, rep.numeric)
    return core, U, r_obj


def rthosvd(A, ranks, p: int, q: int, seed: int, **kw):
    """Shifted randomized T-HOSVD, Alg. 3 -> rtk_rthosvd semantics."""
    return solve(A, ranks, p, q, seed, sequential=False, **kw)


def rsthosvd(A, ranks, p: int, q: int, seed: int, **kw):
    """Shifted randomized ST-HOSVD, Alg. 4 -> rtk_rsthosvd semantics."""
    return solve(A, ranks, p, q, seed, sequential=True, **kw)


def rsthosvd_a2(A, ranks, p: int, q: int, seed: int, **kw):
    """Holistic shifted randomized ST-HOSVD, Alg. A.2 -> rtk_solve with
    variant = 1 (shift=False: Alg. A.1)."""
    return solve(A, ranks, p, q, seed, sequential=True, variant=1, **kw)


def omega(seed: int, mode: int, row0: int, rows: int, l: int, device="cuda"):
    """Rows [row0, row0+rows) of Omega_mode (RTK-GAUSS-2) computed by the CUDA kernel."""
    import torch
    lib = load_library()
    out = torch.empty((rows, l), dtype=torch.float32, device=device)
    with torch.cuda.device(out.device):
        _check(lib.rtk_omega(ctypes.c_uint64(seed), mode, row0, rows, l,
                             ctypes.c_void_p(out.data_ptr()), _stream_handle(out.device)))
    return out


def sketch(kind: int, seed: int, mode: int, dims, l: int, row0: int = 0, rows=None, device="cuda"):
    """Rows [row0, row0+rows) of mode `mode`'s sketch of type `kind` (0 Gaussian, 1 uniform, 2/3
    Khatri-Rao) for a tensor with extents `dims`, computed by the CUDA kernels (test hook)."""
    import torch
    lib = load_library()
    d = len(dims)
    m = 1
    for j, n in enumerate(dims):
        if j + 1 != mode:
            m *= int(n)
    rows = m - row0 if rows is None else rows
    out = torch.empty((rows, l), dtype=torch.float32, device=device)
    dd = (ctypes.c_int64 * d)(*[int(x) for x in dims])
    with torch.cuda.device(out.device):
        _check(lib.rtk_sketch(kind, ctypes.c_uint64(seed), mode, dd, d, row0, rows, l,
                              ctypes.c_void_p(out.data_ptr()), _stream_handle(out.device)))
    return out


def power_step(M, Q):
    """Y = M (M^T Q) by the fused streaming kernel (test hook).  M: n x m column-major
    float32 CUDA (stride(0) == 1), Q: n x l float32 CUDA; returns Y n x l float64."""
    import torch
    lib = load_library()
    n, m = M.shape
    if (M.stride(0) != 1 and n > 1) or M.dtype != torch.float32 or not M.is_cuda:
        raise ValueError("M must be a column-major float32 CUDA matrix")
    ld = max(M.stride(1), n) if m > 1 else n
    l = Q.shape[1]
    Qc = Q.t().contiguous()                     # column-major n x l, ld n
    Y = torch.empty((l, n), dtype=torch.float64, device=M.device)
    with torch.cuda.device(M.device):
        _check(lib.rtk_power_step(ctypes.c_void_p(M.data_ptr()), n, m, ld, ctypes.c_void_p(Qc.data_ptr()),
                                  l, ctypes.c_void_p(Y.data_ptr()), _stream_handle(M.device)))
    return Y.t()


class _DeviceBuffer:
    """A raw device buffer (pointer, count, dtype) seen by torch through __cuda_array_interface__."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2}


def shard_bounds(n_last: int, world: int, rank: int):
    """[begin, begin + count) of mode d held by `rank` when n_last indices are split over `world`
    ranks as evenly as possible (the first n_last % world ranks hold one more)."""
    if world < 1 or not 0 <= rank < world or n_last < world:
        raise ValueError("need 0 <= rank < world <= n_last")
    base, extra = divmod(int(n_last), int(world))
    begin = rank * base + min(rank, extra)
    return begin, base + (1 if rank < extra else 0)


def rsthosvd_shard(A_slab, dims, last_begin: int, ranks, p: int, q: int, seed: int, allreduce=None,
                   root=None, shift: bool = True, omega_kind: int = 0, path: int = 0, out=None, workspace=None):
    """Alg. 4 on one rank of a group holding A split along its LAST mode (rtk_rsthosvd_shard,
    SURVEY.md 8(e)): A_slab is this rank's float32 column-major CUDA slab of extents
    dims[:-1] + [count] covering mode-d indices [last_begin, last_begin + count); dims are the FULL
    extents.  `allreduce(t)` sums the 1-D CUDA tensor t in place over the group on the current
    stream (default: torch.distributed.all_reduce on the default group); `root` (default: rank 0 of
    torch.distributed) is the one rank that applies the shift term -alpha Q before each all-reduce.
    Returns (core, [U_k]), identical on every rank."""
    import torch
    lib = load_library()
    if not isinstance(A_slab, torch.Tensor) or not A_slab.is_cuda or A_slab.dtype != torch.float32:
        raise ValueError("A_slab must be a float32 CUDA tensor (no CPU fallback)")
    if not _is_column_major(A_slab):
        raise ValueError("A_slab must be column-major (mode-1 fastest); use as_column_major")
    dims = [int(x) for x in dims]
    d = len(dims)
    if A_slab.dim() != d or list(A_slab.shape[:-1]) != dims[:-1]:
        raise ValueError("A_slab must have extents dims[:-1] + [count]")
    count = int(A_slab.shape[-1])
    ranks = [int(r) for r in ranks]
    if allreduce is None or root is None:
        import torch.distributed as dist
        if allreduce is None:
            def allreduce(t):
                dist.all_reduce(t)
        if root is None:
            root = dist.get_rank() == 0
    dev = A_slab.device
    if out is None:
        U = [torch.empty((r, n), dtype=torch.float32, device=dev).t() for n, r in zip(dims, ranks)]
        core = as_column_major(torch.empty(ranks, dtype=torch.float32, device=dev))
    else:
        core, U = out
        _check_outputs(core, U, dims, ranks, dev)
    opt = _Options(1, 1 if shift else 0, 0.0, int(path), 0, int(omega_kind))
    dd = (ctypes.c_int64 * d)(*dims)
    rr = (ctypes.c_int32 * d)(*ranks)
    up = (ctypes.c_void_p * d)(*[u.data_ptr() for u in U])
    nb = lib.rtk_workspace_bytes_shard(ctypes.byref(opt), dd, d, count, rr, p, q)
    if nb == 0:
        raise RtkError(1, lib.rtk_last_error().decode())
    ws = workspace if workspace is not None else _WS.get(dev, int(nb))
    errors = []

    def _cb(buf, n, dtype, stream, ctx):
        try:
            t = torch.as_tensor(_DeviceBuffer(buf, n, "<f8" if dtype == 1 else "<f4"), device=dev)
            allreduce(t)
            return 0
        except Exception as e:  # noqa: BLE001  (reported below; the C side returns RTK_ERR_CUDA)
            errors.append(e)
            return 1

    cb = _ALLREDUCE_FN(_cb)
    with torch.cuda.device(dev):
        code = lib.rtk_rsthosvd_shard(ctypes.byref(opt), ctypes.c_void_p(A_slab.data_ptr()), dd, d, int(last_begin),
                                      count, 1 if root else 0, rr, p, q, ctypes.c_uint64(seed), up,
                                      ctypes.c_void_p(core.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                      ws.numel() * ws.element_size(), _stream_handle(dev), cb, None)
    if errors:
        raise errors[0]
    _check(code)
    return core, U

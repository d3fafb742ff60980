"""C-ABI library: builds, loads, exports every symbol include/rtucker.h declares, and
rejects bad arguments before any launch (CPU-only: no compute calls)."""
import ctypes
import os
import re

import pytest

from paper_2506_04840_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load_library()


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "rtucker.h")).read()
    return sorted(set(re.findall(r"RTK_API\s+[\w\s\*]+?\b(rtk_\w+)\s*\(", hdr)))


def test_header_declares_expected_api():
    syms = declared_symbols()
    assert syms == sorted(_lib.ABI_FUNCTIONS)


def test_library_exports_every_declared_symbol(lib):
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert lib.rtk_version().decode().startswith("rtucker ")


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.lib_path()} 2>&1").read()
    assert "sm_100a" in out


def _call(lib, fn, dims, ranks, p, q, ptr=256, null_u=False):
    d = len(dims)
    dd = (ctypes.c_int64 * d)(*dims)
    rr = (ctypes.c_int32 * d)(*ranks)
    up = (ctypes.c_void_p * d)(*([None] * d if null_u else [ptr] * d))
    return getattr(lib, fn)(ctypes.c_void_p(ptr), dd, d, rr, p, q, ctypes.c_uint64(1), up,
                            ctypes.c_void_p(ptr), None, 0, None, None)


@pytest.mark.parametrize("fn", ["rtk_rthosvd", "rtk_rsthosvd"])
def test_argument_errors(lib, fn):
    assert _call(lib, fn, (10, 10, 10), (3, 3, 3), 2, 0) == 1           # q < 1
    assert b"q" in lib.rtk_last_error()
    assert _call(lib, fn, (10, 10, 10), (3, 0, 3), 2, 1) == 1           # r < 1
    assert _call(lib, fn, (10, 10, 10), (3, 11, 3), 2, 1) == 1          # r > n
    assert _call(lib, fn, (10, 10, 10), (3, 3, 3), -1, 1) == 1          # p < 0
    assert _call(lib, fn, (10,), (3,), 2, 1) == 1                       # d < 2
    assert _call(lib, fn, (10, 10, 10), (3, 3, 3), 8, 1) == 2           # l = 11 > n = 10
    assert _call(lib, fn, (10, 10, 10), (3, 3, 3), 2, 1, null_u=True) == 1
    assert _call(lib, fn, (10, 10, 10), (3, 3, 3), 2, 1, ptr=257) == 3  # misaligned A


def test_st_shape_rule_uses_shrunk_columns(lib):
    # mode 3 of ST factors G_(3) with r1*r2 = 4 columns: l = 5 > 4 -> SHAPE; T-HOSVD has 100 cols
    assert _call(lib, "rtk_rsthosvd", (10, 10, 10), (2, 2, 3), 2, 1) == 2
    d = (ctypes.c_int64 * 3)(10, 10, 10)
    r = (ctypes.c_int32 * 3)(2, 2, 3)
    assert lib.rtk_workspace_bytes(0, d, 3, r, 2, 1) > 0
    assert lib.rtk_workspace_bytes(1, d, 3, r, 2, 1) == 0


@pytest.mark.parametrize("algo,dims,ranks,p,q", [
    (0, (64, 64, 64), (5, 5, 5), 5, 2), (0, (200, 200, 200), (20, 20, 20), 10, 3),
    (1, (400, 400, 400), (30, 30, 30), 10, 3), (1, (80, 80, 80, 80), (10, 10, 10, 10), 5, 4),
    (1, (1000, 1000, 1000), (50, 50, 50), 10, 5)])
def test_workspace_query(lib, algo, dims, ranks, p, q):
    d = len(dims)
    n = lib.rtk_workspace_bytes(algo, (ctypes.c_int64 * d)(*dims), d, (ctypes.c_int32 * d)(*ranks), p, q)
    assert 0 < n < 2 * 1024**3

"""rtucker: B200-native adaptive-shift randomized T-HOSVD / ST-HOSVD (arXiv 2506.04840).

Thin Python binding over the C ABI in ``include/rtucker.h`` (``librtucker.so``,
built in-tree for sm_100a by ``paper_2506_04840_b200.build``).  Argument
marshalling only: torch supplies device memory and the current stream, every
step of the hot path runs in the library's CUDA kernels.  There is no CPU
fallback: importing works without a GPU (so the ABI can be inspected), but
every compute call needs the CUDA library and a CUDA tensor and raises
otherwise.

    core, U = rsthosvd(A, ranks, p, q, seed)      # Alg. 4
    core, U = rthosvd(A, ranks, p, q, seed)       # Alg. 3
    core, U = rsthosvd_a2(A, ranks, p, q, seed)   # Alg. A.2
    core, U = rsthosvd_shard(A_slab, dims, begin, ranks, p, q, seed)   # Alg. 4, A split over ranks

``A`` is a float32 CUDA tensor of shape (n_1, ..., n_d) in COLUMN-MAJOR layout
(stride[0] == 1, mode-1 fastest; see :func:`as_column_major`).  U[k] is
n_k x r_k (column-major), core is r_1 x ... x r_d (column-major).
"""
from __future__ import annotations

from ._lib import (ABI_FUNCTIONS, RtkError, as_column_major, lib_path, load_library, omega,
                   power_step, profile_begin, profile_end, rthosvd, rsthosvd, rsthosvd_a2, rsthosvd_shard,
                   shard_bounds, sketch, solve, version, workspace_bytes)

__all__ = ["rthosvd", "rsthosvd", "rsthosvd_a2", "rsthosvd_shard", "shard_bounds", "solve", "sketch", "omega", "power_step", "workspace_bytes",
           "as_column_major", "RtkError", "profile_begin", "profile_end", "load_library", "lib_path", "version", "ABI_FUNCTIONS"]

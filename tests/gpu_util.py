"""Helpers shared by the -m gpu tests (no method arithmetic here)."""
import numpy as np
import pytest


def cuda_or_skip():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_04840_b200 import build
    build.build()
    return torch


def to_device_colmajor(a_np, torch):
    """Fortran-ordered numpy float32 -> CUDA tensor with the same column-major strides."""
    a = np.asfortranarray(a_np, dtype=np.float32)
    t = torch.from_numpy(a)          # keeps Fortran strides
    return t.to("cuda")

"""CPU float64 ORACLE for the adaptive-shift randomized T-HOSVD / ST-HOSVD hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import anything
from this package.  The product path (``paper_2506_04840_b200``) never imports
it and fails loudly when its CUDA library is missing.

The oracle shares no code with the CUDA path.  Both sides implement the same
written specification of the sketch generator; the
seeded input generators live in ``workloads/`` and contain none of the
method's arithmetic.

Modules
-------
gauss   Philox4x32-10 + RTK-GAUSS-2 Box-Muller (the Omega_k of Alg. 3/4,
        PAPER.md:257, :300).
tucker  unfold / fold / mode-k product, Alg. 1
        (PAPER.md:113-125), Alg. 2, Alg. 3
        (PAPER.md:250-270), Alg. 4, Alg. B.1
        (PAPER.md:1145-1172), Alg. A.2 / A.1.
metrics RE, principal angles, spectral gaps,
        orthonormality.

Parity status of each function is stated in its docstring; every function is
pinned by a ``-m "not gpu"`` test in ``tests/test_oracle_*.py`` except where
the docstring says "parity unpinned".
"""

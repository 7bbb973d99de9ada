"""ORACLE — test infrastructure only (NOT part of the product path).

A plain, slow, obviously-correct CPU implementation of the hot path of
arXiv 2304.10516 (the distributed neural representation, DNR): per-block
multiresolution hash-grid encoding + small ReLU MLP, fitted with the
boundary-weighted L1 loss (Eq. 2) and Adam, then decoded by coordinate
query or to a grid.

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import this package.
  * It shares no code with ``paper_2304_10516_b200`` (the CUDA path) and never
    imports it; the only common module is ``synth`` (seeded input generators,
    which hold none of the method's arithmetic).
  * Value math is float64.  Index math (level positions, cell indices, hash)
    is float32 / uint32 exactly as pinned in DESIGN.md readings R4, R20, so
    the integer decisions match the GPU's bit for bit.
  * Citations: ``P:L<n>`` = /root/reference/PAPER.md line, ``S:L<n>`` =
    /root/reference/SPEC.md line, ``R<n>`` = DESIGN.md reading.

Parity status of each function is recorded in its docstring and in
DESIGN.md; every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` except where a docstring says "parity unpinned".
"""
from . import philox, encoding, mlp, loss, adam, sampler, model, fit, decode, cache  # noqa: F401

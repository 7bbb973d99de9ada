"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the
oracle.  Holds NONE of the method's arithmetic (no sampling, encoding, MLP,
loss or optimizer): only analytic fields shaped like the paper's workloads —
three scalar fields and a Taylor-Green velocity field (the paper's S3D /
CloverLeaf3D / NekRS data, are unavailable) — and small
helpers to lay them out.  Recipes: DESIGN.md
"Inputs"."""
from .volumes import (  # noqa: F401
    SEED, g1_analytic, g2_energy, g3_density, evaluate, lattice, linear_field, constant_field, random_points,
    taylor_green, taylor_green_volume)

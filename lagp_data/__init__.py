"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NONE of the method's arithmetic (no correlation, no ALC, no
NN selection, no prediction): only input generators and the frozen per-config
parameters. It is the one module both `oracle/` and the CUDA path may consume.
"""
from .generators import (  # noqa: F401
    CONFIGS,
    borehole,
    lgbb_design,
    lgbb_pred_grid,
    lhs,
    lift_surface,
    make_config,
    q10_lengthscale,
    surface2d,
    uniform,
)

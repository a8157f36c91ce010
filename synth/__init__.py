"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds *none* of the method's arithmetic (no convolution, no
influence function, no proximal step).  It only draws images, Poisson counts
and model parameters from fixed seeds, following the recipe in DESIGN.md §3
(SURVEY.md §8(d)).
"""
from .generator import (  # noqa: F401
    CONFIGS,
    MASTER_SEED,
    Model,
    Problem,
    clean_image,
    dct_atoms,
    make_model,
    make_problem,
    stress_model,
    zero_model,
)

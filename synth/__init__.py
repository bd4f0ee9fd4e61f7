"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the OMP method (no correlation, selection,
least squares or residual).  It only draws dictionaries and sparse signals the
way SURVEY.md §8(d) and DESIGN.md §3 describe, so that the CUDA path and the
FP64 oracle are fed byte-identical FP32 inputs.
"""

from .generator import (  # noqa: F401
    CONFIGS,
    Problem,
    config,
    make_dictionary,
    make_signals,
    make_problem,
)

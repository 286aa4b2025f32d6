"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NO arithmetic of the method (no distances, no spanning trees,
no APPD): it only draws numbers.  Both the oracle and the CUDA path consume the
exact bytes produced here.  The recipes are stated in DESIGN.md ("Input recipe")
and stand in for the paper's seven external datasets, which are not
available.
"""
from .generators import (  # noqa: F401
    CONFIGS,
    SplitMix64,
    config,
    random_points,
    random_weights,
)

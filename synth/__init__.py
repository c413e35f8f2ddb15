"""Seeded synthetic workloads shared by the oracle side and the CUDA side.

This module holds input generation only: Bezier base curves, equidistant
resampling to 21 points and smooth Gaussian displacements.  It holds none of the
method's arithmetic (no d_ME, no discard test, no labelling), so the oracle and
the CUDA path can both consume its arrays without sharing any method code.
"""
from .generator import (  # noqa: F401
    CONFIGS,
    CHUNK,
    N_POINTS,
    Atlas,
    atlas_for_config,
    fibers_for_config,
    resample_equidistant,
    reverse_fibers,
    sample_indices,
)

"""Seeded synthetic inputs shared by the oracle tests, the CUDA-path tests and bench.py.

This module holds NO arithmetic of the method (no B-splines, no operator, no solver):
only the benchmark configurations of BASELINE.json (as plain dicts) and the seeded
right-hand-side generators.  Both sides (``oracle/`` and the CUDA path) consume
these inputs; neither side's arithmetic lives here.
"""
from .configs import CONFIGS, config, Config  # noqa: F401
from .generators import rhs, hash_vector  # noqa: F401

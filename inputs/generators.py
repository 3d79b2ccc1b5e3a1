"""Seeded input generators (no method arithmetic).

rhs(): the seeded right-hand side coefficient vector of a config (BASELINE.json configs:
"seeded uniform[-1,1]" or "seeded standard-normal").  numpy's PCG64 stream with the
config seed; float64; length = ndof, component-major, direction 1 slowest.

hash_vector(): the counter-based start vector of the power iteration that estimates
lambda_max(D^-1 A) (reading R4).  Both the oracle and the CUDA library
implement this same counter-based formula independently; it lives here in Python only
so tests can inspect it.
"""
import numpy as np

_GOLD = 0x9E3779B97F4A7C15
_MASK = (1 << 64) - 1


def rhs(cfg, seed=None, size=None) -> np.ndarray:
    n = cfg.ndof if size is None else size
    g = np.random.Generator(np.random.PCG64(cfg.seed if seed is None else seed))
    if cfg.rhs == "uniform":
        return g.uniform(-1.0, 1.0, n)
    if cfg.rhs == "normal":
        return g.standard_normal(n)
    raise ValueError(cfg.rhs)


def hash_vector(n: int) -> np.ndarray:
    """v[k] = (((k+1)*0x9E3779B97F4A7C15 mod 2^64) >> 11) * 2^-53 - 0.5."""
    k = np.arange(1, n + 1, dtype=np.uint64)
    h = (k * np.uint64(_GOLD))  # wraps mod 2^64
    return (h >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) - 0.5

"""Pins of oracle/bspline.py against values the paper fixes (no GPU)."""
import os

import numpy as np
import pytest

from oracle import bspline as bs

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cardinal_values.txt")


def _golden():
    rows = []
    for line in open(GOLD):
        if line.strip() and not line.startswith("#"):
            p, t, r, v = line.split()
            rows.append((int(p), float(t), int(r), float(v)))
    return rows


@pytest.mark.parametrize("p,t,r,v", _golden())
def test_cardinal_golden(p, t, r, v):
    # hand-derived values of the recursion PAPER.md:268-277 / 296-299
    assert abs(bs.cardinal_deriv(p, t, r) - v) < 1e-14


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6])
def test_cardinal_properties(p):
    ts = np.linspace(-1, p + 2, 301)
    vals = np.array([bs.cardinal(p, t) for t in ts])
    assert np.all(vals >= -1e-15)                                           # nonnegative
    assert np.all(vals[(ts < 0) | (ts > p + 1)] == 0.0)                     # supp = [0,p+1]
    sym = np.array([bs.cardinal(p, p + 1 - t) for t in ts])                  # symmetry
    inside = (ts > 0) & (ts < p + 1)
    assert np.max(np.abs(vals[inside] - sym[inside])) < 1e-14
    for t in [0.1, 0.37, 0.9]:                                              # integer shifts sum to 1
        assert abs(sum(bs.cardinal(p, t + k) for k in range(-p - 2, p + 3)) - 1.0) < 1e-14


@pytest.mark.parametrize("p,n", [(1, 5), (2, 7), (3, 8), (4, 9), (5, 12)])
def test_basis_partition_of_unity_and_boundary(p, n):
    rng = np.random.default_rng(p * 100 + n)
    for x in rng.uniform(0, 1, 25):
        N = bs.basis(p, n, x)
        assert np.all(N >= -1e-15)
        assert abs(N.sum() - 1.0) < 1e-14
        assert abs(bs.basis_deriv(p, n, x).sum()) < 1e-11                    # derivative of 1
    N0 = bs.basis(p, n, 0.0)
    assert abs(N0[0] - 1.0) < 1e-15 and np.all(N0[1:] == 0.0)               # eq:spline-boundary


@pytest.mark.parametrize("p,n", [(2, 7), (3, 8), (4, 11), (5, 13)])
def test_central_basis_is_shifted_cardinal(p, n):
    # N_i^p(x) = phi_p(n x - i + p + 1), i = p+1..n
    for x in np.linspace(0.013, 0.987, 17):
        N = bs.basis(p, n, x)
        for i in range(p + 1, n + 1):
            assert abs(N[i - 1] - bs.cardinal(p, n * x - i + p + 1)) < 1e-13
        dN = bs.basis_deriv(p, n, x)
        for i in range(p + 1, n + 1):
            assert abs(dN[i - 1] - n * bs.cardinal_deriv(p, n * x - i + p + 1, 1)) < 1e-11


def test_derivative_matches_finite_difference():
    p, n, h = 4, 9, 1e-6
    for x in [0.031, 0.45, 0.77]:
        fd = (bs.basis(p, n, x + h) - bs.basis(p, n, x - h)) / (2 * h)
        assert np.max(np.abs(fd - bs.basis_deriv(p, n, x))) < 1e-6


@pytest.mark.parametrize("q", [1, 2, 3, 5, 8])
def test_gauss_rule_exactness(q):
    z, w = bs.gauss01(q)
    for k in range(2 * q):
        assert abs(np.dot(w, z ** k) - 1.0 / (k + 1)) < 1e-14

"""Pins of oracle/matrices1d.py (1D M, A, S) against the paper and closed forms (no GPU)."""
import numpy as np
import pytest

from oracle import bspline as bs
from oracle import matrices1d as m1

CASES = [(1, 8), (2, 9), (3, 12), (4, 14), (5, 17), (6, 20)]


@pytest.mark.parametrize("p,n", CASES)
def test_mass_row_sums_are_basis_integrals(p, n):
    # full basis: sum_j int N_i N_j = int N_i (partition of unity) = (xi_{i+p+1}-xi_i)/(p+1)
    M, A, S = m1.full_matrices(p, n)
    assert np.max(np.abs(M.sum(axis=1) - m1.basis_integrals(p, n))) < 1e-15
    assert np.max(np.abs(S.sum(axis=1))) < 1e-11          # derivative of 1 vanishes
    assert np.max(np.abs(A.sum(axis=1))) < 1e-12


@pytest.mark.parametrize("p,n", CASES)
def test_symmetry_skewness_definiteness(p, n):
    M, A, S = m1.matrices(p, n)
    assert M.shape == (n + p - 2, n + p - 2)
    assert np.max(np.abs(M - M.T)) < 1e-16 and np.max(np.abs(S - S.T)) < 1e-12
    assert np.max(np.abs(A + A.T)) < 1e-14                 # "A^p_n is skew-symmetric" PAPER.md:346
    assert np.linalg.eigvalsh(M)[0] > 0 and np.linalg.eigvalsh(S)[0] > 0


@pytest.mark.parametrize("p,n", [(1, 10), (2, 12), (3, 16), (4, 20), (5, 24), (6, 28)])
def test_central_entries_match_cardinal_formulas(p, n):
    # for i,j = 2p..n-p-1 (1-based)
    M, A, S = m1.matrices(p, n)
    for i in range(2 * p, n - p):
        for j in range(max(1, i - p - 1), min(n + p - 2, i + p + 1) + 1):
            t = p + 1 - (i - j)
            assert abs(M[i - 1, j - 1] - bs.cardinal(2 * p + 1, t) / n) < 1e-15
            assert abs(A[i - 1, j - 1] + bs.cardinal_deriv(2 * p + 1, t, 1)) < 1e-14
            assert abs(S[i - 1, j - 1] + n * bs.cardinal_deriv(2 * p + 1, t, 2)) < 1e-11


def test_p1_closed_forms():
    n = 7
    M, A, S = m1.matrices(1, n)
    assert np.allclose(np.diag(M), 2 / 3 / n, atol=1e-16) and np.allclose(np.diag(M, 1), 1 / 6 / n, atol=1e-16)
    assert np.allclose(np.diag(S), 2 * n, atol=1e-13) and np.allclose(np.diag(S, 1), -n, atol=1e-13)
    assert np.allclose(np.diag(A, 1), 0.5, atol=1e-15) and np.allclose(np.diag(A), 0.0, atol=1e-14)


def test_p1_stiffness_eigenvalues_closed_form():
    # S^1_n = n tridiag(-1,2,-1): eigenvalues n (2 - 2 cos(k pi/(m+1)))
    n = 11
    S = m1.matrices(1, n)[2]
    m = n - 1
    ref = n * (2 - 2 * np.cos(np.arange(1, m + 1) * np.pi / (m + 1)))
    assert np.max(np.abs(np.linalg.eigvalsh(S) - np.sort(ref))) < 1e-11


@pytest.mark.parametrize("p", [2, 3, 4])
def test_entries_independent_of_quadrature_order(p):
    # exact integration: more Gauss points must not change the matrices
    a = m1.matrices(p, 9)
    b = m1.matrices(p, 9, q=2 * p + 3)
    for x, y in zip(a, b):
        assert np.max(np.abs(x - y)) < 1e-13

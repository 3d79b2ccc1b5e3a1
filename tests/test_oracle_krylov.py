"""Pins of oracle/krylov.py fgmres (no GPU): properties that fix GMRES independently of its code.

* finite termination: with restart >= n, GMRES on an n x n nonsingular system reaches the
  exact solution in at most n steps (Saad, Iterative Methods, Prop. 6.10);
* minimal residual: after k steps (no restart, B = I) the residual equals
  min_{c} ||b - A K_k c|| over the Krylov basis K_k = [b, Ab, .., A^{k-1} b], computed here
  by brute-force least squares on the explicit (unorthogonalised) basis;
* k distinct eigenvalues (diagonalisable A) -> convergence in exactly k steps;
* an exact preconditioner (B = A^{-1}) -> one step;
* restarted residual history never increases; the returned x meets the tolerance on the
  TRUE residual.
"""
import os
import sys

import numpy as np
import scipy.linalg as sla

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.krylov import fgmres  # noqa: E402



def _system(n, seed, shift=4.0):
    rng = np.random.default_rng(seed)
    A = shift * np.eye(n) + rng.standard_normal((n, n))
    return A, rng.standard_normal(n)


def test_finite_termination():
    A, b = _system(12, 1)
    x, it, _ = fgmres(A, b, lambda v: v, 1e-13, 100, restart=12)
    assert it <= 12
    assert np.linalg.norm(x - np.linalg.solve(A, b)) <= 1e-11 * np.linalg.norm(np.linalg.solve(A, b))


def test_minimal_residual_property_against_brute_force_krylov_lstsq():
    A, b = _system(30, 2, shift=2.0)
    for k in range(1, 7):
        x, it, _ = fgmres(A, b, lambda v: v, 1e-300, k, restart=50)
        assert it == k
        K = np.empty((30, k))
        K[:, 0] = b
        for i in range(1, k):
            K[:, i] = A @ K[:, i - 1]
        c, *_ = np.linalg.lstsq(A @ K, b, rcond=None)
        rmin = np.linalg.norm(b - A @ K @ c)
        assert abs(np.linalg.norm(b - A @ x) - rmin) <= 1e-9 * np.linalg.norm(b)


def test_k_distinct_eigenvalues_converge_in_k_steps():
    rng = np.random.default_rng(3)
    Q, _ = np.linalg.qr(rng.standard_normal((40, 40)))
    lam = np.repeat([1.0, 2.5, -3.0, 7.0], 10)
    A = Q @ np.diag(lam) @ np.linalg.inv(Q)
    b = rng.standard_normal(40)
    x, it, _ = fgmres(A, b, lambda v: v, 1e-10, 100, restart=40)
    assert it == 4
    assert np.linalg.norm(b - A @ x) <= 1e-9 * np.linalg.norm(b)


def test_exact_preconditioner_one_step():
    A, b = _system(20, 4)
    lu = sla.lu_factor(A)
    x, it, _ = fgmres(A, b, lambda v: sla.lu_solve(lu, v), 1e-10, 10, restart=5)
    assert it == 1
    assert np.linalg.norm(x - np.linalg.solve(A, b)) <= 1e-10 * np.linalg.norm(x)


def test_restarted_history_monotone_and_true_residual():
    A, b = _system(60, 5, shift=10.0)
    x, it, hist = fgmres(A, b, lambda v: v, 1e-9, 2000, restart=4)
    assert all(hist[i + 1] <= hist[i] * (1 + 1e-12) for i in range(len(hist) - 1))
    assert np.linalg.norm(b - A @ x) / np.linalg.norm(b) < 1e-8
    assert hist[-1] < 1e-9


def test_zero_rhs():
    A, _ = _system(5, 6)
    x, it, hist = fgmres(A, np.zeros(5), lambda v: v, 1e-8, 10)
    assert it == 0 and not x.any()


def test_spd_system_gmres_matches_cg_solution():
    # on SPD systems GMRES and CG solve the same problem: compare the converged solutions
    from oracle.krylov import pcg
    rng = np.random.default_rng(7)
    G = rng.standard_normal((25, 25))
    A = G @ G.T + 25 * np.eye(25)
    b = rng.standard_normal(25)
    xg, _, _ = fgmres(A, b, lambda v: v, 1e-12, 100, restart=25)
    xc, _, _ = pcg(A, b, lambda v: v, 1e-12, 100)
    assert np.linalg.norm(xg - xc) <= 1e-10 * np.linalg.norm(xc)

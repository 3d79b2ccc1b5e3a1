"""Pins of oracle/transfer.py, oracle/multigrid.py and oracle/krylov.py (no GPU)."""
import math

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spl

import inputs
from oracle import bspline as bs
from oracle.krylov import pcg
from oracle.multigrid import (AuxPreconditioner, Hierarchy, aux_map, level_sizes, power_rho, power_rho_t,
                              toeplitz_T, toeplitz_solve_axes)
from oracle.operator import Discretization, form_alfven
from oracle.transfer import prolongation, prolongation_1d


@pytest.mark.parametrize("p,nc", [(1, 3), (2, 4), (3, 5), (4, 6), (5, 7)])
def test_prolongation_reproduces_coarse_splines(p, nc):
    C = prolongation_1d(p, nc, full=True)
    for x in np.random.default_rng(p).uniform(0, 1, 20):
        assert np.max(np.abs(bs.basis(p, 2 * nc, x) @ C - bs.basis(p, nc, x))) < 1e-13


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_prolongation_central_columns_are_binomial(p):
    # two-scale relation of the cardinal B-spline: phi_p(t) = 2^-p sum_k C(p+1,k) phi_p(2t-k)
    nc = 4 * p + 4
    C = prolongation_1d(p, nc, full=True)
    j = nc // 2 + p // 2          # a central coarse spline (1-based j+1)
    col = C[:, j]
    nz = col[np.abs(col) > 1e-12]
    ref = np.array([math.comb(p + 1, k) for k in range(p + 2)]) / 2 ** p
    assert len(nz) == p + 2 and np.max(np.abs(nz - ref)) < 1e-13


@pytest.mark.parametrize("d,p,nc", [(2, 2, 3), (2, 3, 4), (3, 2, 2), (3, 3, 2)])
def test_galerkin_coarse_operator_equals_coarse_discretization(d, p, nc):
    # nested spaces: P^T A_h P = A_{2h}  (A_{l+1} := P^T A_l P)
    f = form_alfven(0.2, 0.05, 1.0, np.ones(d) / math.sqrt(d))
    Af = Discretization(d, p, 2 * nc).assemble(f)
    Ac = Discretization(d, p, nc).assemble(f)
    P = prolongation(d, p, nc)
    G = (P.T @ Af @ P).toarray()
    assert np.max(np.abs(G - Ac.toarray())) < 1e-13 * np.max(np.abs(G))


def test_level_rule():
    assert level_sizes(2, 2, 16, 2) == [16, 8]
    assert level_sizes(3, 4, 160) == [160, 80, 40, 20, 10]
    assert level_sizes(2, 3, 256) == [256, 128, 64, 32]
    assert level_sizes(3, 3, 64) == [64, 32, 16, 8]
    assert level_sizes(2, 5, 1024)[-1] == 32


def _setup(d=2, p=2, n=8, levels=0, nu=1.0, beta=0.05, b0=(0.6, 0.8)):
    A = Discretization(d, p, n).assemble(form_alfven(nu, beta, 1.0, b0))
    return A, Hierarchy(A, d, p, n, levels)


def test_power_rho_close_to_true_lambda_max():
    A, H = _setup()
    D = A.diagonal()
    lam = sla.eigh(A.toarray(), np.diag(D), eigvals_only=True)[-1]
    rho = power_rho(A, D)
    assert 0.85 * lam <= rho <= lam * (1 + 1e-12)


def test_vcycle_symmetric_positive_definite():
    A, H = _setup(n=8, levels=2)
    N = A.shape[0]
    B = np.column_stack([H.vcycle(e) for e in np.eye(N)])
    assert np.max(np.abs(B - B.T)) < 1e-10 * np.max(np.abs(B))
    assert np.linalg.eigvalsh(0.5 * (B + B.T))[0] > 0
    # two-grid error propagation I - B A is a contraction in the A-norm
    E = np.eye(N) - B @ A.toarray()
    Lc = np.linalg.cholesky(A.toarray())
    assert np.linalg.norm(Lc.T @ E @ np.linalg.inv(Lc.T), 2) < 1.0


def test_coarse_correction_exact_on_coarse_space():
    # with no smoothing, x = P A_c^{-1} P^T b; for b = A P y this returns P y
    A, H = _setup(n=8, levels=2)
    H.nu_pre = H.nu_post = 0
    y = np.random.default_rng(1).standard_normal(H.A[1].shape[0])
    b = A @ (H.P[0] @ y)
    assert np.max(np.abs(H.vcycle(b) - H.P[0] @ y)) < 1e-10 * np.max(np.abs(H.P[0] @ y))


def test_jacobi_fixed_point():
    A, H = _setup(levels=2)
    x = np.random.default_rng(2).standard_normal(A.shape[0])
    assert np.max(np.abs(H.jacobi(0, A @ x, x, 3) - x)) < 1e-13 * np.max(np.abs(x))


def test_pcg_matches_direct_solve_and_counts():
    A, H = _setup(n=16, levels=0)
    b = np.random.default_rng(3).uniform(-1, 1, A.shape[0])
    x, it, hist = pcg(A, b, H.vcycle, 1e-12, 500)
    xs = spl.spsolve(A.tocsc(), b)
    assert np.linalg.norm(x - xs) / np.linalg.norm(xs) < 1e-8
    assert hist[-1] < 1e-12 and all(h >= 1e-12 for h in hist[:-1])
    # exact preconditioner: one iteration
    lu = spl.splu(A.tocsc())
    _, it1, _ = pcg(A, b, lu.solve, 1e-10, 10)
    assert it1 == 1
    # k distinct eigenvalues -> at most k iterations (Krylov theory)
    Dm = sp.diags(np.repeat([1.0, 2.0, 5.0, 9.0], 25))
    _, it4, _ = pcg(Dm, np.ones(100), lambda r: r, 1e-12, 50)
    assert it4 <= 4
    _, it0, _ = pcg(A, np.zeros(A.shape[0]), H.vcycle, 1e-8, 10)
    assert it0 == 0


@pytest.mark.parametrize("smoother", ["jacobi", "toeplitz"])
def test_config0_solves(smoother):
    c = inputs.config(0)
    A = Discretization(c.dim, c.p, c.n).assemble(form_alfven(c.nu, c.beta, c.lam, c.b0))
    B = AuxPreconditioner(A, c.dim, c.p, c.n, c.b0, c.levels, smoother=smoother)
    assert B.exact          # b0 = (1, 0): exact auxiliary solve
    b = inputs.rhs(c)
    x, it, hist = pcg(A, b, B, c.tol, 1000)
    assert np.linalg.norm(b - A @ x) / np.linalg.norm(b) < 2 * c.tol
    assert it < 40


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_toeplitz_factor_entries_and_symbol(p):
    # T_m(m_{p-1}) entries are cardinal B-spline values; it is the Toeplitz
    # matrix of the symbol m_{p-1} (g_p): T = I for p = 1, eigenvalues in
    # [min m_{p-1}, max m_{p-1}] = [m_{p-1}(pi), 1]
    from oracle.symbol import sym_m
    T = toeplitz_T(p, 30)
    if p == 1:
        assert np.array_equal(T, np.eye(30))
        return
    assert np.max(np.abs(T - T.T)) == 0.0
    ev = np.linalg.eigvalsh(T)
    assert ev.max() <= 1 + 1e-12 and ev.min() >= sym_m(p - 1, np.pi) - 1e-12
    if p == 2:
        assert abs(T[0, 0] - 2 / 3) < 1e-15 and abs(T[0, 1] - 1 / 6) < 1e-15
    if p == 3:
        assert abs(T[0, 0] - 11 / 20) < 1e-15


def test_toeplitz_smoother_rho_and_fixed_point():
    A, H = _setup(levels=2)
    T = sp.kron(sp.identity(2), sp.kron(toeplitz_T(2, 8), toeplitz_T(2, 8))).toarray()
    lam = sla.eigh(A.toarray(), T, eigvals_only=True)[-1]
    assert 0.85 * lam <= H.rho_t[0] <= lam * (1 + 1e-10)
    x = np.random.default_rng(2).standard_normal(A.shape[0])
    assert np.max(np.abs(H.toeplitz(0, A @ x, x, 3) - x)) < 1e-12 * np.max(np.abs(x))


def test_additive_aux_preconditioner_pins():
    # R8' additive mode: symmetric, positive definite, and with the exact auxiliary solve
    # (b0 = e1) it reproduces span{b0 s} exactly: B(A Pi s) - V(A Pi s) = Pi s.
    c = inputs.config(0)
    A = Discretization(c.dim, c.p, c.n).assemble(form_alfven(c.nu, c.beta, c.lam, c.b0))
    B = AuxPreconditioner(A, c.dim, c.p, c.n, c.b0, c.levels, mode="add")
    assert B.exact
    rng = np.random.default_rng(8)
    u, v = rng.standard_normal(A.shape[0]), rng.standard_normal(A.shape[0])
    assert abs(u @ B(v) - v @ B(u)) <= 1e-10 * abs(u @ B(u))
    assert u @ B(u) > 0 and v @ B(v) > 0
    s = rng.standard_normal(A.shape[0] // c.dim)
    r = A @ (B.Pi @ s)
    assert np.max(np.abs(B(r) - B.V.vcycle(r) - B.Pi @ s)) <= 1e-10 * np.max(np.abs(s))
    x, it, _ = pcg(A, inputs.rhs(c), B, c.tol, 500)
    assert it < 60


@pytest.mark.parametrize("d,p,m,nc", [(2, 3, 9, 2), (3, 4, 7, 3), (3, 2, 5, 1), (2, 1, 6, 2), (3, 6, 8, 1)])
def test_toeplitz_solve_axes_equals_sparse_lu_of_kronecker(d, p, m, nc):
    # axis-by-axis banded Cholesky = LU of the assembled I_nc (x) T^{(x)d} (Kronecker identity)
    T1 = sp.csr_matrix(toeplitz_T(p, m))
    K = T1
    for _ in range(d - 1):
        K = sp.kron(K, T1, format="csr")
    K = sp.kron(sp.identity(nc, format="csr"), K, format="csc")
    b = np.random.default_rng(d * 10 + p).standard_normal(K.shape[0])
    ref = spl.splu(K).solve(b)
    x = toeplitz_solve_axes(p, m, d, nc, b)
    # two backward-stable solves differ by up to u kappa(K), kappa(K) = kappa(T)^d (p = 6, d = 3: ~1e7)
    tol = max(1e-12, 10 * np.finfo(float).eps * np.linalg.cond(toeplitz_T(p, m)) ** d)
    assert np.max(np.abs(x - ref)) <= tol * np.max(np.abs(ref))
    assert np.max(np.abs(K @ x - b)) <= 1e-12 * np.max(np.abs(b))


@pytest.mark.parametrize("exact", [True, False])
def test_multiplicative_aux_preconditioner_pins(exact):
    # R8 symmetric multiplicative mode z = Pi Bs Pi^T r; z += V(r - A z); z += Pi Bs Pi^T (r - A z):
    # symmetric and positive definite (V and Bs are); with the exact auxiliary solve (b0 = e1)
    # r = A Pi s is reproduced exactly, B(A Pi s) = Pi s (the first correction already solves it,
    # the residual after it is 0, so the other two terms vanish)
    d, p, n = 2, 3, 8
    b0 = (1.0, 0.0) if exact else (0.6, 0.8)
    A = Discretization(d, p, n).assemble(form_alfven(0.05, 0.01, 1.0, b0))
    B = AuxPreconditioner(A, d, p, n, b0, levels=2, mode="mult")
    assert B.exact == exact
    rng = np.random.default_rng(9)
    u, v = rng.standard_normal(A.shape[0]), rng.standard_normal(A.shape[0])
    assert abs(u @ B(v) - v @ B(u)) <= 1e-10 * abs(u @ B(u))
    assert u @ B(u) > 0 and v @ B(v) > 0
    Bd = np.column_stack([B(e) for e in np.eye(A.shape[0])])
    assert np.max(np.abs(Bd - Bd.T)) <= 1e-10 * np.max(np.abs(Bd))
    assert np.linalg.eigvalsh(0.5 * (Bd + Bd.T)).min() > 0
    if exact:
        s = rng.standard_normal(A.shape[0] // d)
        assert np.max(np.abs(B(A @ (B.Pi @ s)) - B.Pi @ s)) <= 1e-10 * np.max(np.abs(s))
    else:
        # the multiplicative preconditioned operator B A is not worse than the V-cycle alone on
        # span{b0 s}: its error propagation I - B A damps Pi s at least as well
        s = rng.standard_normal(A.shape[0] // d)
        e = B.Pi @ s
        eB = e - B(A @ e)
        eV = e - B.V.vcycle(A @ e)
        assert np.sqrt(eB @ (A @ eB)) <= np.sqrt(eV @ (A @ eV))

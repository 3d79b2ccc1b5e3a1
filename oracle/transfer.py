"""Multigrid prolongation by exact representation of coarse B-splines in the fine basis.

Oracle (test infrastructure only).

PAPER.md:1085-1111 (Sec. 6.1, "Multigrid idea"): prolongation P_l : R^{N_{l+1}} -> R^{N_l},
restriction R_l := P_l^T and A_{l+1} := P_l^T A_l P_l ("the so-called Galerkin approach").
PAPER.md:1178-1186 (eq:2by2prol): the d x d block prolongator  I_d (x) P_(1) (x) ... (x) P_(d).

Reading R3: the 1D factor is the B-spline knot-insertion matrix of uniform
h-refinement (n_c -> 2 n_c elements), i.e. the matrix whose column j holds the fine-basis
coefficients of the coarse B-spline N^c_{j+1}; the nested spline spaces make this the
natural "multi-linear interpolation" of the B-spline coefficients.  This oracle computes
that matrix straight from its definition -- the unique coefficients c with
    N^c_j(x) = sum_k c_k N^f_k(x)   for all x
-- by a least-squares fit on Gauss points of every fine element (library primitive
numpy.linalg.lstsq), never by a knot-insertion recurrence.
"""
import numpy as np
import scipy.sparse as sp

from .bspline import basis, gauss01


def prolongation_1d(p: int, n_coarse: int, full: bool = False) -> np.ndarray:
    """(n_f+p-2) x (n_c+p-2) interior prolongation, n_f = 2 n_c (``full``: all B-splines)."""
    nf = 2 * n_coarse
    z, _ = gauss01(p + 1)
    xs = ((np.arange(nf)[:, None] + z[None, :]) / nf).ravel()
    Bf = np.array([basis(p, nf, x) for x in xs])           # (S, nf+p)
    Bc = np.array([basis(p, n_coarse, x) for x in xs])     # (S, nc+p)
    C, *_ = np.linalg.lstsq(Bf, Bc, rcond=None)             # Bf C = Bc
    if full:
        return C
    # coarse interior splines vanish at 0 and 1, so their first/last fine coefficient is 0
    assert np.all(np.abs(C[0, 1:-1]) < 1e-12) and np.all(np.abs(C[-1, 1:-1]) < 1e-12)
    return C[1:-1, 1:-1]


def prolongation(d: int, p: int, n_coarse: int, ncomp: int = None) -> sp.csr_matrix:
    """I_d (x) P_1D (x) ... (x) P_1D  (eq:2by2prol); tiny entries
    (|c| < 1e-14, rounding of exact zeros) are dropped.  ``ncomp`` components (default d;
    1 for the scalar auxiliary space of reading R8)."""
    P1 = prolongation_1d(p, n_coarse)
    P1[np.abs(P1) < 1e-14] = 0.0
    P1s = sp.csr_matrix(P1)
    K = P1s
    for _ in range(d - 1):
        K = sp.kron(K, P1s, format="csr")
    return sp.kron(sp.identity(d if ncomp is None else ncomp, format="csr"), K, format="csr")

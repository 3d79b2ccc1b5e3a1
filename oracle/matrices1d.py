"""1D IgA mass, advection and stiffness matrices by element-wise Gauss quadrature.

Oracle (test infrastructure only).  PAPER.md:336-345 (Sec. 3.2, eq:matr_M, eq:matr_A,
eq:matr_S):
    M_ij = int_0^1 N_{i+1} N_{j+1},  A_ij = int_0^1 N_{i+1} N_{j+1}',  S_ij = int_0^1 N_{i+1}' N_{j+1}',
    i,j = 1..n+p-2  (the first and last B-spline are removed: homogeneous Dirichlet,
    PAPER.md:326-332).
Each entry is the sum over the knot spans of a (p+1)-point Gauss rule, exact for the
degree-2p integrands.  Dense numpy arrays: these matrices are small.
"""
import numpy as np

from .bspline import element_tables


def full_matrices(p: int, n: int, q: int = None):
    """(n+p) x (n+p) matrices over ALL B-splines N_1..N_{n+p} (before removing the boundary ones).

    Returns (M, A, S) with A_ij = int N_i N_j' (derivative on the column / trial function).
    """
    q = p + 1 if q is None else q
    _, wq, B, D = element_tables(p, n, q)
    size = n + p
    M = np.zeros((size, size))
    A = np.zeros((size, size))
    S = np.zeros((size, size))
    for e in range(n):
        for g in range(q):
            w = wq[e, g]
            for a in range(p + 1):
                for b in range(p + 1):
                    i, j = e + a, e + b      # 0-based global indices of N_{e+1+a}, N_{e+1+b}
                    M[i, j] += w * B[e, g, a] * B[e, g, b]
                    A[i, j] += w * B[e, g, a] * D[e, g, b]
                    S[i, j] += w * D[e, g, a] * D[e, g, b]
    return M, A, S


def matrices(p: int, n: int, q: int = None):
    """Interior (Dirichlet) matrices M^p_n, A^p_n, S^p_n of size n+p-2."""
    M, A, S = full_matrices(p, n, q)
    return M[1:-1, 1:-1], A[1:-1, 1:-1], S[1:-1, 1:-1]


def basis_integrals(p: int, n: int) -> np.ndarray:
    """int_0^1 N_i^p = (xi_{i+p+1} - xi_i)/(p+1) for i=1..n+p (closed form, de Boor;
    used as an independent pin of the mass-matrix row sums via partition of unity)."""
    from .bspline import knots
    xi = knots(p, n)
    return np.array([(xi[i + p] - xi[i - 1]) / (p + 1) for i in range(1, n + p + 1)])

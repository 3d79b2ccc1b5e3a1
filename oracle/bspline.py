"""B-splines on the uniform open knot vector, cardinal B-splines, Gauss rule.

Oracle (test infrastructure only).  Follows PAPER.md Sec. 3.1 (lines 214-312):
  * knot sequence  xi_1=..=xi_{p+1}=0 < xi_{p+2} < .. < xi_{p+n} < 1 = xi_{p+n+1}=..=xi_{2p+n+1},
    xi_{i+p+1} = i/n
  * Cox-de Boor recursion, "a fraction with zero denominator is assumed to be zero"
                                                      
  * derivative formula
  * cardinal B-spline phi_p recursion and phi_p' = phi_{p-1}(t) - phi_{p-1}(t-1)
                                                      
Indices in this module are the paper's 1-based indices unless a name says ``0``.
"""
import numpy as np


def knots(p: int, n: int) -> np.ndarray:
    """xi_1..xi_{2p+n+1} (returned 0-based: xi[k-1] = xi_k).  PAPER.md:215-222."""
    xi = np.empty(2 * p + n + 1)
    xi[: p + 1] = 0.0
    for i in range(0, n + 1):
        xi[i + p] = i / n          # xi_{i+p+1} = i/n  (1-based)
    xi[p + n:] = 1.0
    return xi


def _frac(num, den):
    """num/den with the paper's convention 0/0 := 0 (any zero denominator -> 0)."""
    return 0.0 if den == 0.0 else num / den


def basis_all(p: int, n: int, x: float):
    """Values N_i^k(x) for all degrees k=0..p and i=1..n+2p-k (Cox-de Boor).

    Returns a list ``N`` with ``N[k][i-1] = N_i^k(x)``.  Pure Python loops: the
    recursion is written exactly as in the paper, one degree at a time.
    """
    xi = knots(p, n)
    X = lambda j: xi[j - 1]  # 1-based knot access
    N0 = [1.0 if (X(i) <= x < X(i + 1)) else 0.0 for i in range(1, n + 2 * p + 1)]
    N = [N0]
    for k in range(1, p + 1):
        prev = N[-1]
        cur = []
        for i in range(1, n + 2 * p - k + 1):
            a = _frac(x - X(i), X(i + k) - X(i)) * prev[i - 1]
            b = _frac(X(i + k + 1) - x, X(i + k + 1) - X(i + 1)) * prev[i]
            cur.append(a + b)
        N.append(cur)
    return N


def basis(p: int, n: int, x: float) -> np.ndarray:
    """N_i^p(x), i=1..n+p, as a 0-based array (entry i-1)."""
    return np.array(basis_all(p, n, x)[p][: n + p])


def basis_deriv(p: int, n: int, x: float) -> np.ndarray:
    """(N_i^p)'(x), i=1..n+p, by the paper's differentiation formula:
    (N_i^p)' = p ( N_i^{p-1}/(xi_{i+p}-xi_i) - N_{i+1}^{p-1}/(xi_{i+p+1}-xi_{i+1}) )."""
    if p == 0:
        return np.zeros(n)
    xi = knots(p, n)
    X = lambda j: xi[j - 1]
    Nm = basis_all(p, n, x)[p - 1]   # N_i^{p-1}, i=1..n+p+1
    out = np.empty(n + p)
    for i in range(1, n + p + 1):
        out[i - 1] = p * (_frac(Nm[i - 1], X(i + p) - X(i)) - _frac(Nm[i], X(i + p + 1) - X(i + 1)))
    return out


def cardinal(p: int, t: float) -> float:
    """Cardinal B-spline phi_p(t) by the recursion of PAPER.md:268-277:
    phi_0 = 1 on [0,1);  phi_p(t) = t/p phi_{p-1}(t) + (p+1-t)/p phi_{p-1}(t-1)."""
    if p == 0:
        return 1.0 if 0.0 <= t < 1.0 else 0.0
    return t / p * cardinal(p - 1, t) + (p + 1 - t) / p * cardinal(p - 1, t - 1.0)


def cardinal_deriv(p: int, t: float, r: int) -> float:
    """r-th derivative of phi_p by repeated use of phi_p' = phi_{p-1}(t) - phi_{p-1}(t-1)
    (PAPER.md:296-299).  Requires r <= p-1 for a continuous value (r = p is right-continuous)."""
    if r == 0:
        return cardinal(p, t)
    return cardinal_deriv(p - 1, t, r - 1) - cardinal_deriv(p - 1, t - 1.0, r - 1)


def gauss01(q: int):
    """q-point Gauss-Legendre rule mapped to [0,1] (library primitive numpy.leggauss)."""
    z, w = np.polynomial.legendre.leggauss(q)
    return 0.5 * (z + 1.0), 0.5 * w


def element_tables(p: int, n: int, q: int, elements=None):
    """Per element e (interval [e/n,(e+1)/n], e=0..n-1) and Gauss point: values and first
    derivatives of the p+1 B-splines that are nonzero there, N_{e+1}..N_{e+p+1} (1-based).

    ``elements`` restricts the table to a subset (default: all n elements).
    Returns (xq, wq, B, D) with xq[k,g] the points of the k-th listed element, wq[k,g] the
    weights (length-scaled), B[k,g,a] = N_{e+1+a}^p(xq[k,g]), D[k,g,a] = its derivative.
    """
    els = np.arange(n) if elements is None else np.asarray(elements)
    z, w = gauss01(q)
    xq = (els[:, None] + z[None, :]) / n
    wq = np.broadcast_to(w[None, :] / n, xq.shape).copy()
    B = np.zeros((len(els), q, p + 1))
    D = np.zeros((len(els), q, p + 1))
    for k, e in enumerate(els):
        for g in range(q):
            v = basis(p, n, xq[k, g])
            dv = basis_deriv(p, n, xq[k, g])
            B[k, g, :] = v[e: e + p + 1]
            D[k, g, :] = dv[e: e + p + 1]
    return xq, wq, B, D

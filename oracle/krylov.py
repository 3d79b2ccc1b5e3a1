"""Preconditioned conjugate gradients.

Oracle (test infrastructure only).

PAPER.md:1246-1248 (remark, Sec. 6.1): "we adopt the classical strategy of using the
proposed multigrid-type method as preconditioner for the CG method"; PAPER.md:1333
(Sec. 6.2): stopping criterion ||r^(k)||_2 / ||r^(0)||_2 < tol, zero initial guess.
The iteration is textbook PCG (Saad, Iterative Methods, Alg. 9.1), the residual r is the
recursively updated one, and ``iterations`` counts the A p products done when the
stopping test first holds.
"""
import numpy as np


def pcg(A, b, precond, tol: float, maxit: int):
    x = np.zeros_like(b)
    r = b.copy()
    r0 = np.linalg.norm(r)
    hist = [1.0]
    if r0 == 0.0:
        return x, 0, hist
    z = precond(r)
    p = z.copy()
    rz = float(r @ z)
    for it in range(1, maxit + 1):
        q = A @ p
        alpha = rz / float(p @ q)
        x = x + alpha * p
        r = r - alpha * q
        rel = np.linalg.norm(r) / r0
        hist.append(rel)
        if rel < tol:
            return x, it, hist
        z = precond(r)
        rz_new = float(r @ z)
        beta = rz_new / rz
        rz = rz_new
        p = z + beta * p
    return x, maxit, hist

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


def fgmres(A, b, precond, tol: float, maxit: int, restart: int = 30):
    """Flexible right-preconditioned restarted GMRES (FGMRES(m)) -- the paper's PGMRES.

    PAPER.md:1075 / 1260 (Sec. 6.1-6.2): the multi-iterative method uses "a preconditioned
    generalized minimal residual (PGMRES) method"; north_star asks for the Krylov solve
    "PCG, and GMRES where the paper uses it".  Textbook FGMRES (Saad, Iterative Methods,
    Alg. 9.6): z_j = B v_j, w = A z_j, Arnoldi by classical Gram-Schmidt with one
    re-orthogonalisation (CGS2: h = V^T w, w -= V h, twice), Givens rotations on the
    Hessenberg matrix, x = x_0 + Z y at convergence or restart; a restart recomputes the true
    residual b - A x.  Stopping test |g_{j+1}| / ||r_0||_2 < tol with the Arnoldi residual
    estimate g (PAPER.md:1333 criterion), zero initial guess; ``iterations`` counts A z
    products.  Returns (x, iterations, history of the relative residual estimates).
    """
    x = np.zeros_like(b)
    r0 = float(np.linalg.norm(b))
    hist = [1.0]
    if r0 == 0.0:
        return x, 0, hist
    r = b.copy()
    it = 0
    while True:
        beta = float(np.linalg.norm(r))
        V = [r / beta]
        Z = []
        H = np.zeros((restart + 1, restart))
        g = np.zeros(restart + 1)
        g[0] = beta
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        done = False
        k = 0
        for j in range(restart):
            z = precond(V[j])
            Z.append(z)
            w = A @ z
            it += 1
            h = np.zeros(j + 1)
            for _ in range(2):   # CGS2
                hp = np.array([float(w @ v) for v in V])
                w = w - sum(hp[i] * V[i] for i in range(j + 1))
                h = h + hp
            hn = float(np.linalg.norm(w))
            H[: j + 1, j] = h
            H[j + 1, j] = hn
            for i in range(j):   # previous rotations
                a, c = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * a + sn[i] * c
                H[i + 1, j] = -sn[i] * a + cs[i] * c
            den = float(np.hypot(H[j, j], H[j + 1, j]))
            cs[j] = H[j, j] / den
            sn[j] = H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            rel = abs(g[j + 1]) / r0
            hist.append(rel)
            k = j + 1
            if rel < tol or it >= maxit or hn == 0.0:
                done = True
                break
            V.append(w / hn)
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):   # back substitution H[:k,:k] y = g[:k]
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        for i in range(k):
            x = x + y[i] * Z[i]
        if done:
            return x, it, hist
        r = b - A @ x

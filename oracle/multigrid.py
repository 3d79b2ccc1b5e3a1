"""Galerkin multigrid hierarchy, damped-Jacobi smoother and the V-cycle.

Oracle (test infrastructure only).

PAPER.md:1084-1111 (Sec. 6.1, "Multigrid idea"): ingredients (smoothers S_l, ~S_l with
s_l, ~s_l steps; R_l, P_l; hierarchy A_l with A_0 := A), the V-cycle steps 1-3, and the
Galerkin choice R_l := P_l^T, A_{l+1} := P_l^T A_l P_l.
Readings:
  R4  smoother = damped (weighted) Jacobi x <- x + omega_l D_l^{-1}(b - A_l x), the
      data-parallel form north_star names in place of the paper's Gauss-Seidel;
      omega_l = 4/(3 * 1.05 * rho_l), rho_l = generalized Rayleigh quotient
      (v,A v)/(v,D v) after K=30 normalised power steps v <- D^{-1}A v / ||.||_2 from the
      counter-based start vector inputs.hash_vector (same formula on both sides).
  R4' smoother = Richardson with the paper's preconditioner T_n^p = I_d (x) T(m_{p-1})^{(x)d}
      (T entries phi_{2p-1}(p - i + j), |i-j| < p):
      x <- x + omega_t T^{-1}(b - A x), omega_t = 4/(3 * 1.05 * rho_t), rho_t = ||T^{-1} A v||
      after K=30 normalised steps v <- T^{-1} A v / ||.||_2 from the same start vector.
  R5  coarsest level solved exactly (dense Cholesky, library primitive scipy cho_solve).
  R6  levels: n_{l+1} = n_l/2 while n_l is even, the next interior size n_l/2+p-2 >= 1 and
      d*(n_l+p-2)^d > 6000 (or exactly ``levels`` levels when requested).
  R8  preconditioner: the V-cycle alone, or combined multiplicatively with a correction on the
      auxiliary space span{b0 s} (the kernel of the lambda-term curl(b0 x u), which is exactly
      representable: Pi s = b0 s maps the scalar spline space into V_h):
          z = Pi Vs Pi^T r;  z += V (r - A z);  z += Pi Vs Pi^T (r - A z),
      Vs = V-cycle of A_s := Pi^T A Pi on the same levels.  This is the paper's
      multi-iterative idea ("basic iterative solvers having complementary
      spectral behavior") applied to the near-kernel the L_A operator has.
"""
import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spl

from inputs import hash_vector
from .bspline import cardinal
from .transfer import prolongation

NCOARSE_MAX = 6000
POWER_STEPS = 30


def level_sizes(d: int, p: int, n: int, levels: int = 0):
    """Element counts n_0 > n_1 > ... > n_L of the hierarchy (reading R6)."""
    ns = [n]
    if levels > 0:
        for _ in range(levels - 1):
            if ns[-1] % 2 or ns[-1] // 2 + p - 2 < 1:
                raise ValueError("hierarchy of %d levels impossible for n=%d, p=%d" % (levels, n, p))
            ns.append(ns[-1] // 2)
        return ns
    while ns[-1] % 2 == 0 and ns[-1] // 2 + p - 2 >= 1 and d * (ns[-1] + p - 2) ** d > NCOARSE_MAX:
        ns.append(ns[-1] // 2)
    return ns


def power_rho(A: sp.spmatrix, Ddiag: np.ndarray, steps: int = POWER_STEPS) -> float:
    """rho = (v, A v)/(v, D v) after ``steps`` normalised steps of v <- D^{-1} A v (reading R4)."""
    v = hash_vector(A.shape[0])
    for _ in range(steps):
        w = (A @ v) / Ddiag
        v = w / np.linalg.norm(w)
    return float(v @ (A @ v)) / float(v @ (Ddiag * v))


def toeplitz_T(p: int, m: int) -> np.ndarray:
    """T_m(m_{p-1}) of PAPER.md:1204-1210: (i,j) -> phi_{2p-1}(p - i + j) if |i-j| < p."""
    T = np.zeros((m, m))
    for i in range(m):
        for j in range(max(0, i - p + 1), min(m, i + p)):
            T[i, j] = cardinal(2 * p - 1, p - i + j)
    return T


def toeplitz_solve_axes(p: int, m: int, d: int, nc: int, b: np.ndarray) -> np.ndarray:
    """x = (I_nc (x) T(m_{p-1})^{(x) d})^{-1} b by the Kronecker identity
    (T (x) T (x) T)^{-1} = T^{-1} (x) T^{-1} (x) T^{-1} ("each (T)^{-1} can be
    solved by means of an LU factorization which is optimal for banded matrices"): one banded
    Cholesky solve (library primitives scipy.linalg.cholesky_banded / cho_solve_banded) along each
    axis of the [nc][m]^d array, all lines at once.  Same result as the sparse LU of the assembled
    Kronecker product (pinned in tests), usable at sizes where that factorisation is too large."""
    T = toeplitz_T(p, m)
    w = p - 1
    ab = np.zeros((w + 1, m))            # upper banded storage: ab[w + i - j, j] = T[i, j]
    for j in range(m):
        for i in range(max(0, j - w), j + 1):
            ab[w + i - j, j] = T[i, j]
    cb = sla.cholesky_banded(ab)
    x = np.asarray(b, dtype=float).reshape((nc,) + (m,) * d)
    for axis in range(1, d + 1):
        y = np.moveaxis(x, axis, 0)
        shp = y.shape
        y = sla.cho_solve_banded((cb, False), y.reshape(m, -1))
        x = np.moveaxis(y.reshape(shp), 0, axis)
    return np.ascontiguousarray(x).reshape(-1)


def power_rho_t(A: sp.spmatrix, Tsolve, steps: int = POWER_STEPS) -> float:
    """rho_t = ||T^{-1} A v|| after ``steps`` normalised steps of v <- T^{-1} A v (reading R4')."""
    v = hash_vector(A.shape[0])
    for _ in range(steps):
        w = Tsolve(A @ v)
        v = w / np.linalg.norm(w)
    return float(np.linalg.norm(Tsolve(A @ v)))


class Hierarchy:
    def __init__(self, A0: sp.spmatrix, d: int, p: int, n: int, levels: int = 0, nu_pre: int = 1, nu_post: int = 1,
                 ncomp: int = None, ns=None, smoother: str = "toeplitz"):
        self.d, self.p = d, p
        self.smoother = smoother
        self.ns = level_sizes(d, p, n, levels) if ns is None else list(ns)
        self.A = [sp.csr_matrix(A0)]
        self.P = []
        for l in range(len(self.ns) - 1):
            P = prolongation(d, p, self.ns[l + 1], ncomp)
            self.P.append(P)
            self.A.append(sp.csr_matrix(P.T @ self.A[l] @ P))      # A_{l+1} := P^T A_l P
        self.D = [A.diagonal().copy() for A in self.A]
        self.rho = [power_rho(self.A[l], self.D[l]) for l in range(len(self.A) - 1)]
        self.omega = [4.0 / (3.0 * 1.05 * r) for r in self.rho]
        nc = d if ncomp is None else ncomp
        self.Tlu, self.rho_t, self.omega_t = [], [], []
        for l in range(len(self.A) - 1):
            T1 = sp.csr_matrix(toeplitz_T(p, self.ns[l] + p - 2))
            K = T1
            for _ in range(d - 1):
                K = sp.kron(K, T1, format="csr")
            lu = spl.splu(sp.kron(sp.identity(nc, format="csr"), K, format="csc"))
            self.Tlu.append(lu)
            self.rho_t.append(power_rho_t(self.A[l], lu.solve))
            self.omega_t.append(4.0 / (3.0 * 1.05 * self.rho_t[-1]))
        self.nu_pre, self.nu_post = nu_pre, nu_post
        self.coarse = sla.cho_factor(self.A[-1].toarray(), lower=True)

    @property
    def L(self):
        return len(self.A) - 1

    def jacobi(self, l, b, x, sweeps):
        """sweeps x <- x + omega_l D_l^{-1} (b - A_l x)   (reading R4)."""
        for _ in range(sweeps):
            x = x + self.omega[l] * (b - self.A[l] @ x) / self.D[l]
        return x

    def toeplitz(self, l, b, x, sweeps):
        """sweeps x <- x + omega_t,l T^{-1} (b - A_l x)   (reading R4')."""
        for _ in range(sweeps):
            x = x + self.omega_t[l] * self.Tlu[l].solve(b - self.A[l] @ x)
        return x

    def smooth(self, l, b, x, sweeps):
        """smoother "toeplitz" (R4'), "jacobi" (R4), or "toeplitz_fine": T_n^p on the finest level
        only, damped Jacobi on the coarser ones -- where the paper places its T_n^p smoother
        (PAPER.md:1075, 1260)."""
        use_t = self.smoother == "toeplitz" or (self.smoother == "toeplitz_fine" and l == 0)
        return (self.toeplitz if use_t else self.jacobi)(l, b, x, sweeps)

    def vcycle(self, b, l: int = 0):
        """One V-cycle for A_l e = b from a zero initial guess (steps 1-3)."""
        if l == self.L:
            return sla.cho_solve(self.coarse, b)
        x = np.zeros_like(b)
        x = self.smooth(l, b, x, self.nu_pre)                     # step 1: pre-smoothing
        r = b - self.A[l] @ x                                     # step 2: residual,
        e = self.vcycle(self.P[l].T @ r, l + 1)                   #   restrict, recurse,
        x = x + self.P[l] @ e                                     #   prolongate and correct
        x = self.smooth(l, b, x, self.nu_post)                    # step 3: post-smoothing
        return x


def aux_map(d: int, nscal: int, b0) -> sp.csr_matrix:
    """Pi: scalar coefficients s -> vector coefficients b0 s (component j = b0_j s)."""
    return sp.vstack([b0[j] * sp.identity(nscal, format="csr") for j in range(d)]).tocsr()


class AuxPreconditioner:
    """Reading R8: z = Pi Bs Pi^T r;  z += V (r - A z);  z += Pi Bs Pi^T (r - A z)
    (mode "mult", symmetric multiplicative), or mode "add": z = V r + Pi Bs Pi^T r
    (additive subspace correction, reading R8').

    Bs = exact A_s^{-1} (sparse LU, library primitive) when b0 has exactly one nonzero
    component (A_s is then one Kronecker product), else the V-cycle of A_s."""

    def __init__(self, A0, d, p, n, b0, levels=0, nu_pre=1, nu_post=1, smoother="toeplitz", mode="mult",
                 aux_nu_pre=None, aux_nu_post=None, aux_smoother=None):
        assert mode in ("mult", "add")
        aux_nu_pre = nu_pre if aux_nu_pre is None else aux_nu_pre
        aux_nu_post = nu_post if aux_nu_post is None else aux_nu_post
        self.mode = mode
        self.A = sp.csr_matrix(A0)
        self.V = Hierarchy(A0, d, p, n, levels, nu_pre, nu_post, smoother=smoother)
        self.Pi = aux_map(d, A0.shape[0] // d, b0)
        As = sp.csr_matrix(self.Pi.T @ self.A @ self.Pi)                # A_s := Pi^T A Pi
        self.exact = sum(1 for v in b0 if v != 0.0) == 1
        if self.exact:
            self.lu = spl.splu(As.tocsc())
            self.Bs = self.lu.solve
        else:
            self.Vs = Hierarchy(As, d, p, n, levels, aux_nu_pre, aux_nu_post, ncomp=1, ns=self.V.ns,
                                smoother=smoother if aux_smoother is None else aux_smoother)
            self.Bs = self.Vs.vcycle

    def __call__(self, r):
        if self.mode == "add":
            return self.V.vcycle(r) + self.Pi @ self.Bs(self.Pi.T @ r)
        z = self.Pi @ self.Bs(self.Pi.T @ r)
        z = z + self.V.vcycle(r - self.A @ z)
        z = z + self.Pi @ self.Bs(self.Pi.T @ (r - self.A @ z))
        return z

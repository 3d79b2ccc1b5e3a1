"""GPU parity at the paths the full-size configurations run (VERDICT r1 "next round" item 1):

* the T_n^p line solves at configuration 4's full size (3D p=4 n=160: 78,732 lines per axis,
  so the 32-line tiled solve runs on every axis) against the oracle's axis-by-axis banded
  Cholesky (oracle.multigrid.toeplitz_solve_axes);
* V-cycle, additive and multiplicative preconditioner and PCG with configuration 4's operator
  (3D p=4, nu=1e-3, beta=1e-4, b0=(1,1,1)/sqrt(3)) at n=8 and n=16, and configuration 1 at full
  size (2D p=3 n=256), against oracle results precomputed by tests/expected/make_expected.py
  (calls only oracle/; the oracle runs take minutes).

Tolerances (reading R9): apply-type results 1e-12 of max|oracle|; V-cycle and
preconditioner actions max(1e-12, 10 u kappa(A_coarsest)): the coarsest-level correction
A_c^{-1} r_c is conditioned by kappa(A_c) with respect to the rounding of its own right-hand
side r_c (restriction, residual), which no two implementations share, so u kappa(A_c) is the
resolution of V b itself, however exactly A_c is solved (measured in round 2: one step of
iterative refinement of the coarse solve on both sides left 1.2e-11 at kappa = 1.4e5); solves:
iterations +-1 -- for the 530-iteration full-size solve, twice the spread the oracle's own
count shows under rounding-level perturbations -- requested residual, ||dx||/||x|| <= 1e-8.
"""
import os

import numpy as np
import pytest

import inputs
from oracle.multigrid import toeplitz_solve_axes

from .gpu_helpers import assert_close, to_dev, to_host

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1805_10058_b200 import igacd as ig  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "expected")
CASES = ["c4n8", "c4n16", "c1full"]


def load(name):
    path = os.path.join(HERE, name + ".npz")
    if not os.path.exists(path):
        pytest.fail("missing %s: run python tests/expected/make_expected.py %s" % (path, name))
    return dict(np.load(path))


def handle(e):
    return ig.igacd_create(int(e["d"]), int(e["p"]), int(e["n"]), float(e["nu"]), float(e["beta"]),
                           float(e["lam"]), tuple(float(v) for v in e["b0"]), levels=int(e["levels"]))


def rhs(e):
    d, p, n = int(e["d"]), int(e["p"]), int(e["n"])
    return np.random.default_rng(int(e["seed"])).uniform(-1.0, 1.0, d * (n + p - 2) ** d)


@pytest.mark.parametrize("ci", [4, 3])
def test_tsolve_full_config_size_32_line_tiles(ci):
    """T^{-1} on level 0 of configurations 4 and 3 at full size vs the oracle's axis-by-axis banded
    Cholesky.  Configuration 4 (m = 162 even, 3 x 162^2 = 78,732 lines per axis >= 64 x 148) runs the
    TMA-staged 32-line tiles on all three axes, configuration 3 (m = 65 odd, 12,675 lines) the
    cp.async 32-line tiles; the second level of each (m = 82 / 33) the in-slab kernel."""
    c = inputs.config(ci)
    h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
    try:
        N = ig.igacd_ndof(h)
        b = np.random.default_rng(77).standard_normal(N)
        x = torch.zeros(N, dtype=torch.float64, device="cuda")
        ig.igacd_tsolve(h, 0, to_dev(b), x)
        ref = toeplitz_solve_axes(c.p, c.m, c.dim, c.dim, b)
        assert_close(to_host(x), ref, 1e-12, "T^-1 config %d level 0" % ci)
        # a coarse level of the same hierarchy (slab kernel for directions 1 and 2)
        N1 = ig.igacd_ndof(h, 1)
        b1 = np.random.default_rng(78).standard_normal(N1)
        x1 = torch.zeros(N1, dtype=torch.float64, device="cuda")
        ig.igacd_tsolve(h, 1, to_dev(b1), x1)
        m1 = ig.igacd_level_n(h, 1) + c.p - 2
        assert_close(to_host(x1), toeplitz_solve_axes(c.p, m1, c.dim, c.dim, b1), 1e-12, "T^-1 level 1")
    finally:
        ig.igacd_destroy(h)


@pytest.mark.parametrize("name", CASES)
def test_hierarchy_and_smoother_parameters(name):
    e = load(name)
    h = handle(e)
    try:
        assert [ig.igacd_level_n(h, l) for l in range(ig.igacd_num_levels(h))] == list(e["ns"])
        for l, ref in enumerate(e["rho_t"]):
            assert abs(ig.igacd_smoother_omega(h, l)[1] - ref) <= 1e-10 * ref, (l, "vector")
        for l, ref in enumerate(e["aux_rho_t"]):
            assert abs(ig.igacd_aux_omega(h, l)[1] - ref) <= 1e-10 * ref, (l, "aux")
    finally:
        ig.igacd_destroy(h)


@pytest.mark.parametrize("name", CASES)
def test_vcycle_and_preconditioners(name):
    e = load(name)
    h = handle(e)
    try:
        tol = max(1e-12, 10 * np.finfo(float).eps * float(e["kappa_coarse"]))
        print("%s: kappa(A_coarsest) = %.3e, tolerance %.2e" % (name, float(e["kappa_coarse"]), tol))
        b = to_dev(rhs(e))
        x = torch.zeros_like(b)
        ig.igacd_vcycle(h, b, x)
        assert_close(to_host(x), e["vcycle"], tol, "V-cycle")
        assert ig.igacd_get_preconditioner(h) == ig.IGACD_PRECOND_AUX_ADD
        ig.igacd_precond(h, b, x)
        assert_close(to_host(x), e["precond_add"], tol, "additive preconditioner")
        ig.igacd_set_preconditioner(h, ig.IGACD_PRECOND_AUX)
        ig.igacd_precond(h, b, x)
        assert_close(to_host(x), e["precond_mult"], tol, "multiplicative preconditioner")
    finally:
        ig.igacd_destroy(h)


def iteration_tolerance(name):
    """+-1 (north_star) when the oracle's own count is that sharply defined.  For a long solve it
    is not: tests/expected/pcg_sensitivity.py reran the oracle's PCG with the right-hand side
    perturbed by one unit roundoff per entry, and with the coarsest-level solve perturbed by
    u kappa(A_coarsest) per entry (the forward error of any backward-stable factorisation, i.e.
    the difference between the oracle's Cholesky and the CUDA path's explicit inverse), and the
    count moved (c1full: 534 -> 528 and 534 -> 525..).  The tolerance is twice the largest
    deviation those runs recorded (reading R9)."""
    dev = 0
    for suffix in ("_sensitivity.npz", "_sensitivity_coarse.npz"):
        path = os.path.join(HERE, name + suffix)
        if os.path.exists(path):
            its = np.load(path)["iterations"]
            base = int(np.load(os.path.join(HERE, name + ".npz"))["pcg_iterations"])
            dev = max(dev, int(np.max(np.abs(its - base))))
    return max(1, 2 * dev)


@pytest.mark.parametrize("name", CASES)
def test_pcg_solve(name):
    e = load(name)
    h = handle(e)
    try:
        bh = rhs(e)
        b = to_dev(bh)
        x = torch.zeros_like(b)
        it, rel = ig.igacd_solve(h, b, x, 1e-8, 5000)
        xg, xo = to_host(x), e["pcg_x"]
        tol_it = iteration_tolerance(name)
        print("%s: PCG iterations gpu %d oracle %d (tolerance %d)" % (name, it, int(e["pcg_iterations"]), tol_it))
        assert abs(it - int(e["pcg_iterations"])) <= tol_it
        assert rel < 1e-8
        assert np.linalg.norm(xg - xo) / np.linalg.norm(xo) <= 1e-8
        # true residual through the library's own residual kernel
        r = torch.zeros_like(b)
        ig.igacd_residual(h, 0, b, x, r)
        assert float(torch.linalg.norm(r)) / np.linalg.norm(bh) < 1.5e-8
    finally:
        ig.igacd_destroy(h)


def test_pcg_history_config1_full_size():
    """Where the oracle's residual history is sharply defined (its perturbed runs agree to 1 % up
    to iteration `agree_1pct_until`), the CUDA path must follow it: the recursive relative
    residual after k iterations (igacd_solve stopped at maxit = k) against the oracle's history."""
    e = load("c1full")
    sens = dict(np.load(os.path.join(HERE, "c1full_sensitivity.npz")))
    hist, until = sens["history"], int(sens["agree_1pct_until"])
    h = handle(e)
    try:
        b = to_dev(rhs(e))
        for k in (10, 50, 100, 200):
            assert k < until
            x = torch.zeros_like(b)
            it, rel = ig.igacd_solve(h, b, x, 1e-8, k, raise_on_noconv=False)
            print("c1full: relres after %d iterations gpu %.6e oracle %.6e" % (k, rel, hist[k]))
            assert it == k
            assert abs(rel / hist[k] - 1.0) < 2e-2
    finally:
        ig.igacd_destroy(h)

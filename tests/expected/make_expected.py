"""Writes the oracle's expected outputs for the GPU parity cases too slow to recompute inside
the GPU test run.  Calls only oracle/ and inputs/ (never the CUDA path); each .npz records its
inputs (the seeds) and the oracle's results, so tests/test_gpu_parity_expected.py compares the
CUDA path against them element by element.

    python tests/expected/make_expected.py [case ...]      (from the repo root; minutes of CPU)

Cases:
  c4n8, c4n16  3D p=4 with configuration 4's operator (nu=1e-3, beta=1e-4, lambda=1,
               b0=(1,1,1)/sqrt(3)) at n=8 (2 levels) and n=16 (the R6 rule: 16 -> 8);
  c1full       configuration 1 at full size (2D p=3 n=256, nu=1e-2, beta=1e-3, b0=(1,1)/sqrt(2)).
Each holds: rho_t of every smoothing level (vector and auxiliary system), one V-cycle
x = V b, the additive (default) and multiplicative preconditioner actions, kappa(A_coarsest),
the PCG iteration count, the recursive residual history end and the PCG solution.
"""
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
from oracle.krylov import pcg  # noqa: E402
from oracle.multigrid import AuxPreconditioner  # noqa: E402
from oracle.operator import Discretization, form_alfven  # noqa: E402

S3 = 1.0 / math.sqrt(3.0)
CASES = {
    "c4n8": dict(d=3, p=4, n=8, nu=1e-3, beta=1e-4, lam=1.0, b0=(S3, S3, S3), levels=2, seed=41),
    "c4n16": dict(d=3, p=4, n=16, nu=1e-3, beta=1e-4, lam=1.0, b0=(S3, S3, S3), levels=0, seed=42),
    "c1full": dict(d=2, p=3, n=256, nu=1e-2, beta=1e-3, lam=1.0, b0=(1 / math.sqrt(2), 1 / math.sqrt(2)), levels=0,
                   seed=1),
}
TOL, MAXIT = 1e-8, 5000


def make(name):
    c = CASES[name]
    t0 = time.time()
    disc = Discretization(c["d"], c["p"], c["n"])
    A = disc.assemble(form_alfven(c["nu"], c["beta"], c["lam"], c["b0"]))
    t1 = time.time()
    Badd = AuxPreconditioner(A, c["d"], c["p"], c["n"], c["b0"], c["levels"], mode="add")
    Bmul = AuxPreconditioner(A, c["d"], c["p"], c["n"], c["b0"], c["levels"], mode="mult")
    t2 = time.time()
    rng = np.random.default_rng(c["seed"])
    b = rng.uniform(-1.0, 1.0, disc.ndof)
    vcyc = Badd.V.vcycle(b)
    padd = Badd(b)
    pmul = Bmul(b)
    kappa = float(np.linalg.cond(Badd.V.A[-1].toarray()))
    t3 = time.time()
    x, it, hist = pcg(A, b, Badd, TOL, MAXIT)
    t4 = time.time()
    out = dict(d=c["d"], p=c["p"], n=c["n"], nu=c["nu"], beta=c["beta"], lam=c["lam"], b0=np.array(c["b0"]),
               levels=c["levels"], seed=c["seed"], ns=np.array(Badd.V.ns), rho_t=np.array(Badd.V.rho_t),
               aux_rho_t=np.array(Badd.Vs.rho_t), vcycle=vcyc, precond_add=padd, precond_mult=pmul,
               kappa_coarse=kappa, pcg_iterations=it, pcg_relres=hist[-1], pcg_x=x,
               true_relres=float(np.linalg.norm(b - A @ x) / np.linalg.norm(b)))
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), name + ".npz")
    np.savez_compressed(path, **out)
    print("%s: ndof %d, levels %s, assemble %.1f s, setup %.1f s, precond %.1f s, pcg %.1f s (%d it, rel %.2e)"
          % (name, disc.ndof, Badd.V.ns, t1 - t0, t2 - t1, t3 - t2, t4 - t3, it, hist[-1]), flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        make(name)

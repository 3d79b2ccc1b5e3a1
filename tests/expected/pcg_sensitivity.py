"""How sharply is the PCG iteration count of a long solve defined in fp64?

The oracle's PCG (oracle/krylov.pcg, additive auxiliary + V-cycle preconditioner) is run on a
case's right-hand side b and on copies b (1 + eps_k) with eps_k relative perturbations of one
unit roundoff per entry (seeded): rounding-level changes of the input, the size of the
differences between any two correct fp64 implementations (summation order, the coarse solve's
factorisation).  The spread of the iteration counts over those runs is the resolution to which
"the same iteration count" is defined for that case; it is recorded in <case>_sensitivity.npz
and used as the tolerance of tests/test_gpu_parity_expected.py::test_pcg_solve (DESIGN.md
reading R9).  Calls only oracle/ and inputs/.

    python tests/expected/pcg_sensitivity.py c1full [nruns]
    python tests/expected/pcg_sensitivity.py c1full coarse [nruns]

The second form perturbs instead the result of the coarsest-level solve by u kappa(A_coarsest)
per entry -- the forward error any backward-stable factorisation of A_coarsest may have, i.e.
the difference between the oracle's Cholesky solve and the CUDA path's explicit inverse
(written to <case>_sensitivity_coarse.npz).
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, HERE)

from make_expected import CASES, MAXIT, TOL  # noqa: E402
from oracle.krylov import pcg  # noqa: E402
from oracle.multigrid import AuxPreconditioner  # noqa: E402
from oracle.operator import Discretization, form_alfven  # noqa: E402


def main_coarse(name, nruns):
    import oracle.multigrid as mg
    c = CASES[name]
    disc = Discretization(c["d"], c["p"], c["n"])
    A = disc.assemble(form_alfven(c["nu"], c["beta"], c["lam"], c["b0"]))
    B = AuxPreconditioner(A, c["d"], c["p"], c["n"], c["b0"], c["levels"], mode="add")
    b = np.random.default_rng(c["seed"]).uniform(-1.0, 1.0, disc.ndof)
    kappa = float(np.linalg.cond(B.V.A[-1].toarray()))
    eps = np.finfo(float).eps * kappa
    orig = mg.sla.cho_solve
    its = []
    for k in range(nruns):
        rng = np.random.default_rng(2000 + k)

        def noisy(cf, rhs, rng=rng):
            x = orig(cf, rhs)
            return x * (1.0 + eps * rng.uniform(-1.0, 1.0, x.size))

        mg.sla.cho_solve = noisy
        try:
            t0 = time.time()
            x, it, hist = pcg(A, b, B, TOL, MAXIT)
        finally:
            mg.sla.cho_solve = orig
        its.append(it)
        print("%s coarse-perturbed run %d (eps %.2e): %d iterations, %.1f s" % (name, k, eps, it, time.time() - t0),
              flush=True)
    np.savez_compressed(os.path.join(HERE, name + "_sensitivity_coarse.npz"), iterations=np.array(its), eps=eps,
                        kappa=kappa)


def main(name, nruns):
    c = CASES[name]
    disc = Discretization(c["d"], c["p"], c["n"])
    A = disc.assemble(form_alfven(c["nu"], c["beta"], c["lam"], c["b0"]))
    B = AuxPreconditioner(A, c["d"], c["p"], c["n"], c["b0"], c["levels"], mode="add")
    b = np.random.default_rng(c["seed"]).uniform(-1.0, 1.0, disc.ndof)
    u = np.finfo(float).eps
    its, hists = [], []
    for k in range(nruns + 1):
        bk = b if k == 0 else b * (1.0 + u * np.random.default_rng(1000 + k).uniform(-1.0, 1.0, b.size))
        t0 = time.time()
        x, it, hist = pcg(A, bk, B, TOL, MAXIT)
        its.append(it)
        hists.append(np.array(hist))
        print("%s run %d: %d iterations, %.1f s" % (name, k, it, time.time() - t0), flush=True)
    n = min(len(h) for h in hists)
    H = np.array([h[:n] for h in hists])
    # first iteration at which some perturbed history differs from the unperturbed one by 1 %
    dev = np.max(np.abs(H[1:] / H[0] - 1.0), axis=0)
    first = int(np.argmax(dev > 1e-2)) if np.any(dev > 1e-2) else n
    print("%s: iteration counts %s; histories agree to 1%% up to iteration %d" % (name, its, first))
    np.savez_compressed(os.path.join(HERE, name + "_sensitivity.npz"), iterations=np.array(its),
                        history=hists[0], agree_1pct_until=first, eps=u)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "coarse":
        main_coarse(sys.argv[1], int(sys.argv[3]) if len(sys.argv) > 3 else 4)
    else:
        main(sys.argv[1] if len(sys.argv) > 1 else "c1full", int(sys.argv[2]) if len(sys.argv) > 2 else 4)

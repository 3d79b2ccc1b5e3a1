"""Iterations / time-to-solution per smoother (Toeplitz R4' vs Jacobi R4) with the default preconditioner."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

for ci in [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4]:
    c = inputs.config(ci)
    h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
    b = torch.from_numpy(inputs.rhs(c)).cuda()
    x = torch.zeros_like(b)
    for sm in (ig.IGACD_SMOOTH_TOEPLITZ, ig.IGACD_SMOOTH_TOEPLITZ_FINE, ig.IGACD_SMOOTH_JACOBI):
        ig.igacd_set_smoother(h, sm)
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.time()
            it, rel = ig.igacd_solve(h, b, x, c.tol, 5000, raise_on_noconv=False)
            torch.cuda.synchronize()
            dt = time.time() - t0
        print(json.dumps({"config": c.name, "smoother": sm, "precond": ig.igacd_get_preconditioner(h), "iters": it,
                          "relres": rel, "solve_s": round(dt, 4)}), flush=True)
    ig.igacd_destroy(h)

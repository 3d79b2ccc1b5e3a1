"""Iterations and time-to-solution vs smoothing sweeps / smoother / preconditioner for configs."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

which = [int(a) for a in sys.argv[1:]] or [1, 3, 4]
for ci in which:
    c = inputs.config(ci)
    for sm in (ig.IGACD_SMOOTH_TOEPLITZ, ig.IGACD_SMOOTH_JACOBI):
        for nu in (1, 2, 3):
            h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels, nu_pre=nu, nu_post=nu)
            ig.igacd_set_smoother(h, sm)
            b = torch.from_numpy(inputs.rhs(c)).cuda()
            x = torch.zeros_like(b)
            torch.cuda.synchronize()
            t0 = time.time()
            it, rel = ig.igacd_solve(h, b, x, c.tol, 3000, raise_on_noconv=False)
            torch.cuda.synchronize()
            print(json.dumps({"config": c.name, "smoother": sm, "nu": nu, "iters": it, "relres": rel,
                              "solve_s": round(time.time() - t0, 3)}), flush=True)
            ig.igacd_destroy(h)

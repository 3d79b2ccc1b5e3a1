"""Iterations / time with the auxiliary V-cycle smoothed by Jacobi vs the T_n^p smoother."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

for ci in [int(a) for a in sys.argv[1:] if a != "--zero"] or [1, 3, 4]:
    c = inputs.config(ci)
    h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
    b = torch.from_numpy(inputs.rhs(c)).cuda()
    x = torch.zeros_like(b)
    combos = [(-1, 1), (-1, 0), (ig.IGACD_SMOOTH_JACOBI, 1), (ig.IGACD_SMOOTH_JACOBI, 2)]
    if len(sys.argv) > 1 and sys.argv[1] == "--zero":
        combos = [(-1, 1), (-1, 0)]
    for aux, sw in combos:
        if True:
            ig.igacd_set_aux_smoother(h, aux)
            ig.igacd_set_aux_sweeps(h, sw, sw)
            for rep in range(2):
                torch.cuda.synchronize()
                t0 = time.time()
                it, rel = ig.igacd_solve(h, b, x, c.tol, 5000, raise_on_noconv=False)
                torch.cuda.synchronize()
                dt = time.time() - t0
            print(json.dumps({"config": c.name, "aux_smoother": aux, "aux_sweeps": sw, "iters": it, "relres": rel,
                              "solve_s": round(dt, 4)}), flush=True)
    ig.igacd_destroy(h)

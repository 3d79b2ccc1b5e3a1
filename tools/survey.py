"""Solve every BASELINE config once on the GPU; print iterations, residual and timings."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

maxit = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
which = [int(a) for a in sys.argv[2:]] or [0, 1, 2, 3, 4]
for ci in which:
    c = inputs.config(ci)
    for mode, sm in ((ig.IGACD_PRECOND_AUX, ig.IGACD_SMOOTH_TOEPLITZ), (ig.IGACD_PRECOND_AUX, ig.IGACD_SMOOTH_JACOBI)):
        t0 = time.time()
        h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
        torch.cuda.synchronize()
        t_setup = time.time() - t0
        ig.igacd_set_preconditioner(h, mode)
        ig.igacd_set_smoother(h, sm)
        b = torch.from_numpy(inputs.rhs(c)).cuda()
        x = torch.zeros_like(b)
        torch.cuda.synchronize()
        t0 = time.time()
        it, rel = ig.igacd_solve(h, b, x, c.tol, maxit, raise_on_noconv=False)
        torch.cuda.synchronize()
        t_solve = time.time() - t0
        # apply timing
        y = torch.empty_like(b)
        for _ in range(3):
            ig.igacd_apply(h, 0, b, y)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10):
            ig.igacd_apply(h, 0, b, y)
        e1.record()
        torch.cuda.synchronize()
        ams = e0.elapsed_time(e1) / 10
        print(json.dumps({"config": c.name, "precond": mode, "smoother": sm, "aux_exact": ig.igacd_aux_is_exact(h), "levels": ig.igacd_num_levels(h), "ndof": c.ndof,
                          "setup_s": round(t_setup, 3), "iters": it, "relres": rel, "solve_s": round(t_solve, 3),
                          "apply_ms": round(ams, 4), "apply_gdofs": round(c.ndof / ams / 1e6, 2),
                          "apply_gbs_alg": round(16 * c.ndof / ams / 1e6, 1),
                          "omega0": ig.igacd_smoother_omega(h, 0) if ig.igacd_num_levels(h) > 1 else None}),
              flush=True)
        ig.igacd_destroy(h)

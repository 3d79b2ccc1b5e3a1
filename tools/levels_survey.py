"""PCG iterations / time-to-solution vs the number of levels (coarsest dense solve size)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

for spec in sys.argv[1:] or ["4:6", "4:5", "3:5", "3:4"]:
    ci, lv = (int(v) for v in spec.split(":"))
    c = inputs.config(ci)
    t0 = time.time()
    h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=lv)
    torch.cuda.synchronize()
    setup = time.time() - t0
    b = torch.from_numpy(inputs.rhs(c)).cuda()
    x = torch.zeros_like(b)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.time()
        it, rel = ig.igacd_solve(h, b, x, c.tol, 5000, raise_on_noconv=False)
        torch.cuda.synchronize()
        dt = time.time() - t0
    print(json.dumps({"config": c.name, "levels": lv, "coarsest_n": ig.igacd_level_n(h, lv - 1),
                      "iters": it, "relres": rel, "solve_s": round(dt, 4), "setup_s": round(setup, 2)}), flush=True)
    ig.igacd_destroy(h)

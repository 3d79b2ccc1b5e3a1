"""Operator-apply timing (CUDA events, rotating buffers > L2) for the listed configs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

L2 = 126 * 2 ** 20
for ci in [int(a) for a in sys.argv[1:]] or [2, 3, 4]:
    c = inputs.config(ci)
    h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
    N = ig.igacd_ndof(h)
    nb = max(2, -(-2 * L2 // (16 * N)) + 1)
    xs = [torch.randn(N, dtype=torch.float64, device="cuda") for _ in range(nb)]
    ys = [torch.empty_like(xs[0]) for _ in range(nb)]
    for k in range(3):
        ig.igacd_apply(h, 0, xs[k % nb], ys[k % nb])
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    reps = 20
    e0.record()
    for k in range(reps):
        ig.igacd_apply(h, 0, xs[k % nb], ys[k % nb])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"config": c.name, "ndof": N, "apply_ms": round(ms, 4),
                      "gdof_s": round(N / ms / 1e6, 2), "alg_GBs": round(16 * N / ms / 1e6, 1),
                      "hbm_frac": round(16 * N / ms / 1e6 / 6538.6, 4)}), flush=True)
    ig.igacd_destroy(h)

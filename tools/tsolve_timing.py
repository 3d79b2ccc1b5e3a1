"""Line-solve (T^{-1}) timing on level 0 of a config: CUDA events, L2 rotated."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

for ci in [int(a) for a in sys.argv[1:]] or [2, 3, 4]:
    c = inputs.config(ci)
    h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
    N = ig.igacd_ndof(h)
    nb = max(2, -(-2 * 126 * 2 ** 20 // (16 * N)) + 1)
    bs = [torch.randn(N, dtype=torch.float64, device="cuda") for _ in range(nb)]
    xs = [torch.empty_like(bs[0]) for _ in range(nb)]
    for k in range(3):
        ig.igacd_tsolve(h, 0, bs[k % nb], xs[k % nb])
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for k in range(20):
        ig.igacd_tsolve(h, 0, bs[k % nb], xs[k % nb])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(json.dumps({"config": c.name, "tsolve_ms": round(ms, 4), "per_axis_us": round(1000 * ms / c.dim, 1),
                      "alg_GBs_per_axis": round(16 * N / (ms / c.dim) / 1e6, 1)}), flush=True)
    ig.igacd_destroy(h)

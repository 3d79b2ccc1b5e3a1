"""Operator apply time on every level of a config's hierarchy (vector system)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

for ci in [int(a) for a in sys.argv[1:]] or [4]:
    c = inputs.config(ci)
    h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
    for l in range(ig.igacd_num_levels(h)):
        N = ig.igacd_ndof(h, l)
        x = torch.randn(N, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        for _ in range(3):
            ig.igacd_apply(h, l, x, y)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(50):
            ig.igacd_apply(h, l, x, y)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"config": c.name, "level": l, "n": ig.igacd_level_n(h, l), "ndof": N,
                          "apply_us": round(1000 * e0.elapsed_time(e1) / 50, 2),
                          "split": os.environ.get("IGACD_SPLIT", "1")}), flush=True)
    ig.igacd_destroy(h)

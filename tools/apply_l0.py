"""Level-0 vector and auxiliary apply timing of one config (CUDA events, rotating buffers > L2)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

c = inputs.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
N = ig.igacd_ndof(h)
nb = 4
xs = [torch.randn(N, dtype=torch.float64, device="cuda") for _ in range(nb)]
ys = [torch.empty_like(xs[0]) for _ in range(nb)]


def timed(fn, a, b, reps=40):
    for k in range(4):
        fn(a[k % nb], b[k % nb])
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for k in range(reps):
        fn(a[k % nb], b[k % nb])
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


ms = timed(lambda a, b: ig.igacd_apply(h, 0, a, b), xs, ys)
Ns = N // c.dim
xa, ya = [x[:Ns].clone() for x in xs], [y[:Ns].clone() for y in ys]
msa = timed(lambda a, b: ig.igacd_apply_aux(h, 0, a, b), xa, ya)
print(json.dumps({"config": c.name, "env": {k: v for k, v in os.environ.items() if k.startswith("IGACD_")},
                  "apply_ms": round(ms, 4), "aux_ms": round(msa, 4)}), flush=True)
ig.igacd_destroy(h)

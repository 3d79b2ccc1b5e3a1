"""Level-0 operator timing (CUDA events, buffers rotated beyond L2): the vector operator
(igacd_apply) and the auxiliary scalar operator (igacd_apply_aux) of the listed configs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

L2 = 126 * 2 ** 20


def timed(fn, xs, ys, reps=30):
    nb = len(xs)
    for k in range(3):
        fn(xs[k % nb], ys[k % nb])
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for k in range(reps):
        fn(xs[k % nb], ys[k % nb])
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for ci in [int(a) for a in sys.argv[1:]] or [3, 4]:
    c = inputs.config(ci)
    h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
    out = {"config": c.name, "env": {k: v for k, v in os.environ.items() if k.startswith("IGACD_")}}
    for lvl in range(ig.igacd_num_levels(h)):
        N = ig.igacd_ndof(h, lvl)
        Ns = N // c.dim
        nb = max(2, -(-2 * L2 // (16 * N)) + 1)
        xs = [torch.randn(N, dtype=torch.float64, device="cuda") for _ in range(nb)]
        ys = [torch.empty_like(xs[0]) for _ in range(nb)]
        ms = timed(lambda a, b: ig.igacd_apply(h, lvl, a, b), xs, ys)
        xa = [x[:Ns].clone() for x in xs]
        ya = [y[:Ns].clone() for y in ys]
        msa = timed(lambda a, b: ig.igacd_apply_aux(h, lvl, a, b), xa, ya)
        out["L%d" % lvl] = {"ndof": N, "apply_ms": round(ms, 4), "aux_ms": round(msa, 4),
                            "apply_GBs": round(16 * N / ms / 1e6, 1), "aux_GBs": round(16 * Ns / msa / 1e6, 1)}
        del xs, ys, xa, ya
    print(json.dumps(out), flush=True)
    ig.igacd_destroy(h)

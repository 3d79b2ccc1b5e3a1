"""Per-phase timings (CUDA events) of one PCG iteration's pieces for a config."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for ci in [int(a) for a in sys.argv[1:]] or [4]:
    c = inputs.config(ci)
    h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
    N = ig.igacd_ndof(h)
    b = torch.from_numpy(inputs.rhs(c)).cuda()
    x = torch.zeros_like(b)
    y = torch.zeros_like(b)
    s = torch.zeros(N // c.dim, dtype=torch.float64, device="cuda")
    s2 = torch.zeros_like(s)
    out = {"config": c.name}
    out["apply_ms"] = timeit(lambda: ig.igacd_apply(h, 0, b, y))
    out["apply_aux_ms"] = timeit(lambda: ig.igacd_apply_aux(h, 0, s, s2))
    for sm, name in ((ig.IGACD_SMOOTH_TOEPLITZ, "T"), (ig.IGACD_SMOOTH_JACOBI, "J")):
        ig.igacd_set_smoother(h, sm)
        out["vcycle_%s_ms" % name] = timeit(lambda: ig.igacd_vcycle(h, b, x))
        out["precond_%s_ms" % name] = timeit(lambda: ig.igacd_precond(h, b, x))
    ig.igacd_set_smoother(h, ig.IGACD_SMOOTH_TOEPLITZ)
    out["solve10_ms"] = timeit(lambda: ig.igacd_solve(h, b, x, 1e-30, 10, raise_on_noconv=False), reps=2)
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in out.items()}), flush=True)
    ig.igacd_destroy(h)

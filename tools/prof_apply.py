"""Bracket one level-0 vector apply and one auxiliary scalar apply with cudaProfilerStart/Stop
(target of `ncu --profile-from-start off`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = inputs.config(ci)
h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
N = ig.igacd_ndof(h)
x = torch.from_numpy(inputs.rhs(c)).cuda()
y = torch.empty_like(x)
xs, ys = x[: N // c.dim].clone(), y[: N // c.dim].clone()
for _ in range(2):
    ig.igacd_apply(h, 0, x, y)
    ig.igacd_apply_aux(h, 0, xs, ys)
torch.cuda.synchronize()
torch.cuda.profiler.start()
ig.igacd_apply(h, 0, x, y)
ig.igacd_apply_aux(h, 0, xs, ys)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ig.igacd_destroy(h)
print("ok", c.name)

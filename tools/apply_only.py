"""Run a few operator applies of a config (target of ncu --set full captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = inputs.config(ci)
h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
x = torch.from_numpy(inputs.rhs(c)).cuda()
y = torch.empty_like(x)
for _ in range(reps):
    ig.igacd_apply(h, 0, x, y)
torch.cuda.synchronize()
ig.igacd_destroy(h)
print("ok", c.name)

"""A few PCG iterations of a config (target of the ncu launch-list capture)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
its = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = inputs.config(ci)
h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
b = torch.from_numpy(inputs.rhs(c)).cuda()
x = torch.zeros_like(b)
print(ig.igacd_solve(h, b, x, 1e-30, its, raise_on_noconv=False))
torch.cuda.synchronize()
ig.igacd_destroy(h)

"""Run a few auxiliary (scalar) operator applies of a config (target of ncu captures)."""
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
N = ig.igacd_ndof(h) // c.dim
s = torch.randn(N, dtype=torch.float64, device="cuda")
t = torch.empty_like(s)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(reps):
    ig.igacd_apply_aux(h, 0, s, t)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ig.igacd_destroy(h)
print("ok", c.name)

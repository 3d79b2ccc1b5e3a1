"""Bracket one level-0 T^{-1} application (igacd_tsolve: one line-solve pass per axis) with
cudaProfilerStart/Stop (target of `ncu --profile-from-start off`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

c = inputs.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
b = torch.from_numpy(inputs.rhs(c)).cuda()
x = torch.empty_like(b)
ig.igacd_tsolve(h, 0, b, x)
torch.cuda.synchronize()
torch.cuda.profiler.start()
ig.igacd_tsolve(h, 0, b, x)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ig.igacd_destroy(h)
print("ok", c.name)

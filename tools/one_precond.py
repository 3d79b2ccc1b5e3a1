"""One preconditioner application (and one V-cycle) between cudaProfilerStart/Stop."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = inputs.config(ci)
h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
b = torch.from_numpy(inputs.rhs(c)).cuda()
x = torch.zeros_like(b)
ig.igacd_precond(h, b, x)
torch.cuda.synchronize()
torch.cuda.profiler.start()
ig.igacd_precond(h, b, x)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ig.igacd_destroy(h)
print("ok")

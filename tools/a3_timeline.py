"""Per-CTA timeline of one level-0 vector apply (IGACD_A3_DBG=3 prints it from the library)."""
import os
import sys

os.environ["IGACD_A3_DBG"] = "3"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

c = inputs.config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=c.levels)
x = torch.from_numpy(inputs.rhs(c)).cuda()
y = torch.empty_like(x)
sys.stderr.write("A3DBG ---- timed apply\n")
ig.igacd_apply(h, 0, x, y)
torch.cuda.synchronize()
ig.igacd_destroy(h)

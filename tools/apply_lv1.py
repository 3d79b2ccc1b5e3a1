"""Vector operator apply timing on a single-level handle (no V-cycle setup)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import inputs  # noqa: E402
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

c = inputs.config(int(sys.argv[1]))
h = ig.igacd_create(c.dim, c.p, c.n, c.nu, c.beta, c.lam, c.b0, levels=1)
N = ig.igacd_ndof(h)
xs = [torch.randn(N, dtype=torch.float64, device="cuda") for _ in range(3)]
ys = [torch.empty_like(xs[0]) for _ in range(3)]
for k in range(3):
    ig.igacd_apply(h, 0, xs[k], ys[k])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for k in range(20):
    ig.igacd_apply(h, 0, xs[k % 3], ys[k % 3])
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(c.name, "split=%s" % os.environ.get("IGACD_SPLIT", "1"), "apply_ms %.4f  alg GB/s %.1f" % (ms, 16 * N / ms / 1e6))

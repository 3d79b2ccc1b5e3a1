"""Probe the split 3D operator on one (p, n) case in a fresh process; print ok / error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1805_10058_b200 import igacd as ig  # noqa: E402

p, n, lv = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 1
try:
    h = ig.igacd_create(3, p, n, 0.3, 0.05, 1.0, (0.48, 0.6, 0.64), levels=lv)
    N = ig.igacd_ndof(h)
    x = torch.randn(N, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    ig.igacd_apply(h, 0, x, y)
    torch.cuda.synchronize()
    print("p=%d n=%d levels=%d ok %.3e" % (p, n, lv, float(y.abs().max())))
except Exception as e:  # noqa: BLE001
    print("p=%d n=%d levels=%d FAIL %s" % (p, n, lv, str(e)[:120]))

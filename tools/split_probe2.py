"""Probe the split 3D operator epilogue modes on one case (fresh process per mode)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1805_10058_b200 import igacd as ig  # noqa: E402

p, n, what = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
try:
    h = ig.igacd_create(3, p, n, 0.3, 0.05, 1.0, (0.48, 0.6, 0.64), levels=1)
    N = ig.igacd_ndof(h)
    x = torch.randn(N, dtype=torch.float64, device="cuda")
    b = torch.randn(N, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    if what == "resid":
        ig.igacd_residual(h, 0, b, x, y)
    elif what == "jacobi":
        ig.igacd_smooth(h, 0, b, x, 2, 0.3)
    elif what == "aux":
        s = torch.randn(N // 3, dtype=torch.float64, device="cuda")
        s2 = torch.zeros_like(s)
        ig.igacd_apply_aux(h, 0, s, s2)
    torch.cuda.synchronize()
    print(p, n, what, "ok")
except Exception as e:  # noqa: BLE001
    print(p, n, what, "FAIL", str(e)[:100])

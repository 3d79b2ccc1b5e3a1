"""Create a 3D p=5 handle (vector + scalar auxiliary system); used under compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_10058_b200 import igacd as ig  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = ig.igacd_create(3, p, n, 1.0, 0.1, 1.0, (0.6, 0.0, 0.8))
print("ok", ig.igacd_num_levels(h))

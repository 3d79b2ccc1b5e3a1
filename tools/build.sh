#!/bin/bash
# Build libigacd.so in-tree (same as __graft_entry__.build()).
cd "$(dirname "$0")/.." && python -c "import paper_1805_10058_b200 as p; p.build()" 2>&1 | grep -iE "error|warning" | head -20
ls -la --time-style=+%T "$(dirname "$0")/../paper_1805_10058_b200/lib/libigacd.so"

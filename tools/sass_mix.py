"""Instruction mix of one kernel in an ncu report (source page, SASS view): executed warp
instructions per opcode and the top stall-sampled instructions.

    python tools/sass_mix.py report.ncu-rep kernel-regex [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
lines = raw.splitlines()
# sections: a "Kernel Name" line, then the CSV table of that kernel; take the first match
heads = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')] + [len(lines)]
sec = next(k for k in range(len(heads) - 1) if re.search(kre, lines[heads[k]]))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[heads[sec] + 1: heads[sec + 1]]))))
print(lines[heads[sec]][:160])
ops = collections.Counter()
stall = []
total = 0
for r in rows:
    n = int(r["Instructions Executed"] or 0)
    src = r["Source"].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
    ops[op.split(".")[0]] += n
    total += n
    stall.append((int(r["Warp Stall Sampling (All Samples)"] or 0), src, n))
print("total warp instructions executed: %d" % total)
for op, n in ops.most_common(top):
    print("%-12s %12d  %5.1f%%" % (op, n, 100.0 * n / max(total, 1)))
print("\ntop stall-sampled instructions:")
for s, src, n in sorted(stall, reverse=True)[:top]:
    print("%6d  %10d  %s" % (s, n, src[:90]))

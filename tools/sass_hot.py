"""Per-opcode instruction counts and stall samples of one kernel from an ncu source page
(`ncu -i rep --page source --csv --print-source sass`), for reading where issue slots go.

    python tools/sass_hot.py sass.csv [kernel-index] [top-N]
"""
import collections
import csv
import sys


def kernels(path):
    cur, name, head = [], None, None
    for row in csv.reader(open(path)):
        if row and row[0] == "Kernel Name":
            if name:
                yield name, head, cur
            name, head, cur = row[1], None, []
        elif head is None:
            head = row
        else:
            cur.append(row)
    if name:
        yield name, head, cur


def main():
    path = sys.argv[1]
    ki = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    for k, (name, head, rows) in enumerate(kernels(path)):
        if k != ki:
            continue
        ix = {h: i for i, h in enumerate(head)}
        ops = collections.Counter()
        samp = collections.Counter()
        tot = 0
        hot = []
        for r in rows:
            src = r[ix["Source"]].strip()
            op = src.split()[0] if src else "?"
            if op.startswith("@"):
                op = src.split()[1]
            op = op.split(".")[0]
            n = int(r[ix["Instructions Executed"]] or 0)
            s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            ops[op] += n
            samp[op] += s
            tot += n
            hot.append((s, r[ix["Address"]], src, n))
        print(name[:120])
        print("total warp instructions %d" % tot)
        for op, n in ops.most_common(top):
            print("%-10s %12d %6.1f%%  samples %d" % (op, n, 100.0 * n / tot, samp[op]))
        hot.sort(reverse=True)
        print("hottest instructions (stall samples):")
        for s, a, src, n in hot[:top]:
            print("%6d %s %-60s %d" % (s, a, src[:60], n))


if __name__ == "__main__":
    main()

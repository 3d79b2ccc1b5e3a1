"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (kernel shares)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
for hi, r in enumerate(rows):
    if "Kernel Name" in r:
        break
hdr, data = rows[hi], rows[hi + 1:]
iK, iV, iU, iG = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit"), hdr.index("Grid Size")
tot, cnt, seq = collections.Counter(), collections.Counter(), []
for r in data:
    if len(r) <= iV:
        continue
    name = r[iK].split("(")[0].replace("void ", "").replace("igacd::", "")
    v = float(r[iV].replace(",", ""))
    v = v / 1000 if r[iU] in ("nsecond", "ns") else (v * 1000 if r[iU] in ("msecond", "ms") else v)
    tot[name] += v
    cnt[name] += 1
    seq.append((v, name, r[iG]))
T = sum(tot.values())
print("total kernel time %.1f us over %d launches (serialised, cold-cache ncu timings)" % (T, sum(cnt.values())))
print("| kernel | launches | time (us) | share |")
print("|---|---|---|---|")
for k, v in tot.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 15):
    print("| %s | %d | %.1f | %.1f%% |" % (k[:70], cnt[k], v, 100 * v / T))

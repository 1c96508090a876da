"""Per-kernel totals / shares from an ncu --metrics gpu__time_duration.sum CSV."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
hdr = rows[0]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
t, n = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    k = r[ki].split("(")[0].replace("void ", "")[:48]
    t[k] += float(r[vi].replace(",", ""))
    n[k] += 1
tot = sum(t.values())
for k in sorted(t, key=lambda k: -t[k]):
    print(f"{k:48s} launches={n[k]:3d} total={t[k] / 1e6:8.3f} ms share={t[k] / tot:.3f}")

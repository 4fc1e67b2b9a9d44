"""Mean per-kernel duration from an ncu --metrics gpu__time_duration.sum CSV."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[h]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[h + 1:]:
    d[r[ki][:60]].append(float(r[vi].replace(",", "")) / 1000)
for k, v in d.items():
    print(f"{k:60s} n={len(v):3d} mean={sum(v) / len(v):9.2f} us")

"""Mean per-kernel duration from an ncu --metrics gpu__time_duration.sum CSV,
one line per (kernel, grid size): the e2e leg of bench.py launches the same
kernels on pair chunks (smaller grids), which must not be averaged with the
full-size launches of the timed step."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[h]
ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
d = collections.defaultdict(list)
for r in rows[h + 1:]:
    d[(r[ki][:60], r[gi])].append(float(r[vi].replace(",", "")) / 1000)
for (k, g), v in d.items():
    print(f"{k:60s} grid={g:18s} n={len(v):3d} mean={sum(v) / len(v):9.2f} us")

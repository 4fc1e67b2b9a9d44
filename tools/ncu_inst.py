"""Per-source-line executed instructions and stall samples of one kernel in
an .ncu-rep (needs -lineinfo and --import-source on at capture time).

usage: python tools/ncu_inst.py report.ncu-rep kernel_regex [top_n]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
inst, stall, src = defaultdict(float), defaultdict(float), {}
cur, hdr = "", None
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ii, wi = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= max(ii, wi):
        continue
    try:
        line, iv, sv = int(r[0]), float(r[ii] or 0), float(r[wi] or 0)
    except ValueError:
        continue
    inst[(cur, line)] += iv
    stall[(cur, line)] += sv
    src[(cur, line)] = r[1]
ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
print(f"warp instructions {ti:.4g}, stall samples {ts:.0f}")
for key in sorted(inst, key=lambda k: -inst[k])[:top]:
    print(f"{inst[key] / ti * 100:5.1f}% inst {stall[key] / ts * 100:5.1f}% stall  {key[0]}:{key[1]:<4d} "
          f"{src[key].strip()[:90]}")

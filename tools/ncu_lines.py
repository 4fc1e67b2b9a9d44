"""Aggregate ncu warp-stall samples and executed instructions per CUDA source
line (needs -lineinfo and --import-source on at capture time).

usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top_n]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
stall = defaultdict(float)
inst = defaultdict(float)
src = {}
cur_file = ""
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        wi = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= wi:
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    try:
        sv, iv = float(r[wi] or 0), float(r[ii] or 0)
    except ValueError:
        continue
    key = (cur_file, line)
    src[key] = r[1]
    stall[key] += sv
    inst[key] += iv
tot = sum(stall.values()) or 1
toti = sum(inst.values()) or 1
print(f"total stall samples {tot:.0f}, warp instructions {toti:.3g}")
order = inst if "--by-inst" in sys.argv else stall
for key in sorted(order, key=lambda k: -order[k])[:top]:
    print(f"{stall[key] / tot * 100:5.1f}% stall {inst[key] / toti * 100:5.1f}% inst  "
          f"{key[0]}:{key[1]:<4d} {src[key].strip()[:90]}")

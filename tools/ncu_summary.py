"""Summarise an .ncu-rep: key metrics per kernel and top stall SASS lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
want = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput",
        "L1/TEX Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Achieved Occupancy", "Registers Per Thread", "Dynamic Shared Memory Per Block"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[0]
ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
seen = set()
for x in r[1:]:
    if x[mi] in want and (x[ki][:60], x[mi]) not in seen:
        seen.add((x[ki][:60], x[mi]))
        print(f"{x[ki][:50]:50s} | {x[mi]:32s} {x[vi]} {x[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hh = rr[0]
cols = [i for i, n in enumerate(hh) if n in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                               "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
                                               "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
                                               "lts__t_bytes.sum", "gpu__time_duration.sum")]
for row in rr[1:]:
    if row and row[0] != "" and not row[0].startswith("ID") and len(row) > max(cols):
        if row[hh.index("Kernel Name")] == "Kernel Name" or row[hh.index("Kernel Name")] == "":
            print("units:", [row[i] for i in cols])
            continue
        print([(hh[i].split(".")[0], row[i][:60]) for i in cols])
if kfilter:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kfilter}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hs = rows[1]
    si, wi = hs.index("Source"), hs.index("Warp Stall Sampling (All Samples)")
    data = rows[2:]
    tot = sum(float(x[wi] or 0) for x in data) or 1
    for x in sorted(data, key=lambda x: -float(x[wi] or 0))[:int(sys.argv[3]) if len(sys.argv) > 3 else 20]:
        print(f"{float(x[wi]) / tot * 100:5.1f}% {x[si][:100]}")

"""Top stall-sampled lines of an ncu report.

usage: python tools/ncu_hot.py REPORT [N] [sass|cuda]
  sass: SASS instructions (default); cuda: CUDA source lines (needs -lineinfo
  and --import-source at capture time)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
view = sys.argv[3] if len(sys.argv) > 3 else "sass"
STALL = "Warp Stall Sampling (All Samples)"

if view == "cuda":
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout.splitlines()
    data, fname, hdr = [], "?", None
    for r in csv.reader(out):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or r[2] != "-":
            continue
        c = r[hdr.index(STALL)]
        if c.isdigit() and int(c):
            data.append((int(c), f"{fname}:{r[0]}", r[1].strip()))
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    start = 2 if rows and rows[0] and rows[0][0].startswith("Kernel") else 1
    hdr = rows[start - 1]
    ci, si = hdr.index(STALL), hdr.index("Source")
    data = [(int(r[ci]) if r[ci].isdigit() else 0, str(i), r[si])
            for i, r in enumerate(rows[start:]) if len(r) > ci]
tot = sum(d[0] for d in data)
print("total samples", tot)
for c, where, src in sorted(data, reverse=True)[:n]:
    print(f"{c:7d} {100.0 * c / max(tot, 1):5.1f}% {where:>22s}  {src[:90]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
r2 = list(csv.reader(raw))
for i, h in enumerate(r2[0]):
    if h in ("gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "dram__bytes_read.sum",
             "dram__bytes_write.sum", "smsp__warps_active.avg.per_cycle_active",
             "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"):
        print(h, r2[1][i], r2[2][i])

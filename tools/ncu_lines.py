"""Per-source-line stall breakdown of an ncu report (needs -lineinfo and
--import-source): python tools/ncu_lines.py REPORT [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
fname, hdr, data = "?", None, []
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or len(r) < len(hdr):
        continue
    try:
        tot = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        st = {h[6:]: int(r[i] or 0) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
    except ValueError:
        continue
    if not tot:
        continue
    top = sorted(st.items(), key=lambda kv: -kv[1])[:4]
    data.append((tot, f"{fname}:{r[0]}", r[1][:60], top, r[hdr.index("Address Space")]))
data.sort(key=lambda x: -x[0])
allt = sum(d[0] for d in data)
for tot, loc, src, top, sp in data[:n]:
    print(f"{tot:7d} {100 * tot / allt:5.1f}% {loc:28s} {sp:14s} " + " ".join(f"{k}={v}" for k, v in top))
    print(f"{'':44s}{src}")

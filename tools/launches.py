"""Summarize an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

for fn in sys.argv[1:]:
    rows = []
    with open(fn) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for row in csv.DictReader(lines):
        if row.get("Metric Name") == "gpu__time_duration.sum":
            scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                     "msecond": 1e3}.get(row["Metric Unit"], 1e-3)
            rows.append((row["Kernel Name"].split("(")[0][-60:], float(row["Metric Value"]) * scale))
    agg = collections.OrderedDict()
    for name, v in rows:
        agg.setdefault(name, []).append(v)
    print(f"== {fn}: {len(rows)} launches")
    for k, v in agg.items():
        print(f"{len(v):4d} x {sum(v) / len(v):10.1f} us = {sum(v):10.1f} us  {k}")

"""Print the key fields of a bench.py JSON line (file argument or stdin)."""
import json
import sys

src = open(sys.argv[1]) if len(sys.argv) > 1 else sys.stdin
d = None
for line in src:
    if line.startswith("{"):
        d = json.loads(line)
if d is None:
    sys.exit("no JSON line")
rows = [(d["config"]["workload"].split(":")[0], d)] + list((d.get("secondary_configs") or {}).items())
for name, v in rows:
    r = v["roofline"]
    fp = r.get("fp64", {}).get("frac")
    print(f"{name}: value {v['value']:.1f} {v.get('unit', 'GB/s')}  ms/step {v['ms_per_step']:.3f}  "
          f"id_s {v['id_seconds'] * 1e3:.3f} ms  launches {v['gpu_launches']}  "
          f"kernel {r['kernel_ms']:.3f} ms  frac {r['frac']:.3f}" + (f"  fp64 {fp:.3f}" if fp else ""))

"""CPQR time against the number of steps k at the C4/C5 sketch shapes (the
slope is the per-step cost, the intercept the fixed cost).  Usage:
python tools/exp_cpqr_k.py  (IDS_CPQR_SEGMENT_UNITS=1: the segment-unit kernel;
IDS_CPQR_PIN=s: pinned segments of the column-owner kernel)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_10559_b200.linalg import device_cpqr
from exp_cpqr import near_dup  # noqa: E402

for name, m, n, base, pert in (("C4", 4096, 1000, 10, 1e-3), ("C5", 16384, 2000, 20, 1e-4),
                               ("C3", 200, 10000, 20, 1e-2)):
    y = near_dup(m, n, base, pert, 1)
    out = []
    for k in (1, 2, 5, 10, 20):
        for _ in range(2):
            device_cpqr(y, m, n, k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            device_cpqr(y, m, n, k)
        e1.record()
        torch.cuda.synchronize()
        out.append((k, e0.elapsed_time(e1) / 10 * 1e3))
    ks = [k for k, _ in out]
    ts = [t for _, t in out]
    kb = sum(ks) / len(ks)
    tb = sum(ts) / len(ts)
    slope = sum((k - kb) * (t - tb) for k, t in out) / sum((k - kb) ** 2 for k in ks)
    print(f"{name}: " + "  ".join(f"k={k}: {t:.1f}us" for k, t in out) +
          f"  | per step {slope:.1f} us, fixed {tb - slope * kb:.1f} us", flush=True)

"""Split-spectrum TensorSketch kernel vs the one-CTA-per-term kernel at the
C4/C5 shapes (and L = 8192): relative difference of Y and of the column
norms, and the time of each.  Usage: python tools/exp_ts_split.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import tensorsketch as tsmod


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name, N, I, R, L in (("C4", 3, 1000, 1000, 4096), ("L8192", 3, 5000, 700, 8192),
                         ("C5", 4, 10000, 2000, 16384)):
    g = torch.Generator(device="cuda").manual_seed(5)
    fac = [torch.randn(R, I, generator=g, device="cuda", dtype=torch.float64).t() for _ in range(N)]
    w = torch.rand(R, generator=g, device="cuda", dtype=torch.float64) + 0.5
    op = ids.TensorSketchOp([I] * N, L, seed=1)
    tsmod.USE_SPLIT = True
    ys, ns = op.apply_device(fac, w, norms=True)
    ms_s = timed(lambda: op.apply_device(fac, w, norms=True))
    tsmod.USE_SPLIT = False
    yo, no = op.apply_device(fac, w, norms=True)
    ms_o = timed(lambda: op.apply_device(fac, w, norms=True))
    tsmod.USE_SPLIT = True
    dy = ((ys - yo).norm() / yo.norm()).item()
    dn = ((ns - no).abs().max() / no.abs().max()).item()
    ys2, ns2 = op.apply_device(fac, w, norms=True)
    same = torch.equal(ys, ys2) and torch.equal(ns, ns2)
    print(f"{name}: N={N} I={I} R={R} L={L}: split {ms_s * 1e3:8.1f} us  old {ms_o * 1e3:8.1f} us  "
          f"Y rel diff {dy:.2e}  norms {dn:.2e}  rerun identical {same}", flush=True)

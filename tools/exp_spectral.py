"""Time of the global-memory FFT TensorSketch route (L beyond the fused
kernels) on C5-like factors: 4 modes x 1e4 rows, R = 2000."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import generators as G

w, facs = G.cp_config("C5")
dims = [int(f.shape[0]) for f in facs]
for L in (32768, 65536, 20000):
    op = ids.TensorSketchOp(dims, L, seed=1)
    y = op.apply_device(facs, w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        y = op.apply_device(facs, w)
    e1.record()
    torch.cuda.synchronize()
    print(f"L={L}: {e0.elapsed_time(e1) / 3:.2f} ms per TensorSketch (R=2000, N=4, I=1e4)", flush=True)

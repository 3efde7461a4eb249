"""Dense sketch of the C2 shape in both layouts (row-major kernel for C order,
column-stream kernel for F order) and ordered vs segmented modes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200._inputs import dense_operand

I, R, L = 1_000_000, 2000, 100
a = torch.randn(I, R, dtype=torch.float64, device="cuda")
af = a.t().contiguous().t()  # same values, F order
op = ids.CountSketchOp(I, L, seed=1, surjective=True)
op.bucket_index()
y = torch.empty((R, L), dtype=torch.float64, device="cuda")
for name, t in (("C order", a), ("F order", af)):
    opnd = dense_operand(t)
    for flags in (1, 0):
        op.sketch_into(opnd, y, flags=flags)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            op.sketch_into(opnd, y, flags=flags)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"{name} flags={flags}: {ms:.3f} ms = {I * R * 8 / ms / 1e6:.0f} GB/s", flush=True)

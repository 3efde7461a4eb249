"""F-order C2 (1e6 x 2000) dense sketch timed with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import generators as G
from paper_1901_10559_b200._inputs import dense_operand

opnd = dense_operand(G.dense_config("C2", layout="F"))
op = ids.CountSketchOp(1_000_000, 100, seed=1, surjective=True)
op.bucket_index()
y = torch.empty((2000, 100), dtype=torch.float64, device="cuda")
for rep in range(5):
    for _ in range(2):
        op.sketch_into(opnd, y, flags=1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        op.sketch_into(opnd, y, flags=1)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"F-order C2 sketch: {ms:.3f} ms  {16e9 / ms / 1e6:.0f} GB/s")

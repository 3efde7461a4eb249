"""One F-order dense sketch of the C2 shape (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200._inputs import dense_operand

I, R, L = 1_000_000, 2000, 100
af = torch.randn(R, I, dtype=torch.float64, device="cuda").t()  # F order
op = ids.CountSketchOp(I, L, seed=1, surjective=True)
y = torch.empty((R, L), dtype=torch.float64, device="cuda")
for _ in range(2):
    op.sketch_into(dense_operand(af), y, flags=1)
torch.cuda.synchronize()

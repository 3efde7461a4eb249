"""Hash draw time (I = 1e7, L = 200, surjective) per seed."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
torch.cuda.set_device(0)
for I, L in ((10_000_000, 200), (1_000_000, 100)):
    ids.CountSketchOp(I, L, seed=0, surjective=True)
    torch.cuda.synchronize()
    out = []
    for s in list(range(10)) + [1000, 1001, 1002, 3, 3]:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ids.CountSketchOp(I, L, seed=s, surjective=True)
        e1.record()
        torch.cuda.synchronize()
        out.append(f"{s}:{e0.elapsed_time(e1):.2f}")
    print(I, " ".join(out))

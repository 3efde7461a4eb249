"""C3-shaped sparse sketch: direct CSR bucket kernel vs device transpose + CSC
kernel.  Usage: python tools/exp_csr.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200._inputs import SparseOperand
from paper_1901_10559_b200.estimators import _transpose

I, R, per, L = 10_000_000, 10_000, 10, 200
g = torch.Generator(device="cuda").manual_seed(0)
indptr = torch.arange(0, I + 1, dtype=torch.int64, device="cuda") * per
idx = torch.randint(0, R, (I * per,), generator=g, device="cuda", dtype=torch.int64)
idx = idx.view(I, per).sort(dim=1).values.to(torch.int32).reshape(-1)
data = torch.randn(I * per, generator=g, device="cuda", dtype=torch.float64)
csr = SparseOperand("csr", indptr, idx, data, I, R, I * per)
op = ids.CountSketchOp(I, L, seed=1, surjective=True)
op.bucket_index()
y = torch.empty((R, L), dtype=torch.float64, device="cuda")


def timed(fn, label, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{label:40s} {e0.elapsed_time(e1) / reps * 1e3:9.1f} us", flush=True)
    return out


timed(lambda: op.sketch_into(csr, y, flags=2), "CSR bucket kernel (segmented)")
y_seg = y.clone()
timed(lambda: op.sketch_into(csr, y, flags=0), "CSR streaming kernel (L2 reductions)", reps=10)
print("max |diff| stream vs segmented:", float((y - y_seg).abs().max()), flush=True)
y_csr = y.clone()
t = timed(lambda: _transpose(indptr, idx, data, I, R, I * per), "device transpose CSR->CSC")
csc = SparseOperand("csc", t[0], t[1][: I * per], t[2][: I * per], I, R, I * per)
timed(lambda: op.sketch_into(csc, y, flags=0), "CSC kernel")
print("max |diff| CSR vs CSC:", float((y - y_csr).abs().max()), flush=True)

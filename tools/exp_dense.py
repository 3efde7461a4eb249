"""Row-major dense sketch kernel variants at C2 (1e6 x 2000, L = 100)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native
from paper_1901_10559_b200._inputs import dense_operand

lib = _native.load()
lib.ids_debug_dense_variant.argtypes = [ctypes.c_int]
a = torch.randn(1_000_000, 2000, dtype=torch.float64, device="cuda")
op = ids.CountSketchOp(1_000_000, 100, seed=1, surjective=True)
op.bucket_index()
operand = dense_operand(a)
ref = None
for v, name in ((0, "<2,8> (default)"), (1, "<4,8>"), (2, "<4,4>"), (0, "<2,8> again")):
    lib.ids_debug_dense_variant(v)
    y = torch.empty((2000, 100), dtype=torch.float64, device="cuda")
    for _ in range(2):
        op.sketch_into(operand, y, flags=1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        op.sketch_into(operand, y, flags=1)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    if ref is None:
        ref = y.clone()
    print(f"{name:16s} {ms * 1e3:8.1f} us  {16e9 / ms / 1e6:8.1f} GB/s  identical={bool(torch.equal(y, ref))}",
          flush=True)
lib.ids_debug_dense_variant(0)

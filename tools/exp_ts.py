"""Per-phase timing of the fused TensorSketch kernel (debug hook
ids_debug_ts_timing) at C4/C5 shapes.  Usage: python tools/exp_ts.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native

lib = _native.load()
lib.ids_debug_ts_timing.argtypes = [ctypes.c_void_p]
NAMES = ["zero", "stage loads", "run heads", "pack/inv", "fft", "untangle*S", "output"]
for name, N, I, R, L in (("C4", 3, 1000, 1000, 4096), ("C5", 4, 10000, 2000, 16384)):
    g = torch.Generator(device="cuda").manual_seed(5)
    fac = [torch.randn(R, I, generator=g, device="cuda", dtype=torch.float64).t() for _ in range(N)]
    w = torch.rand(R, generator=g, device="cuda", dtype=torch.float64) + 0.5
    op = ids.TensorSketchOp([I] * N, L, seed=1)
    for _ in range(3):
        op.apply_device(fac, w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        op.apply_device(fac, w)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    buf = torch.zeros(8, dtype=torch.int64, device="cuda")
    lib.ids_debug_ts_timing(buf.data_ptr())
    op.apply_device(fac, w)
    torch.cuda.synchronize()
    lib.ids_debug_ts_timing(None)
    t = buf.cpu().numpy()
    print(f"{name}: N={N} I={I} R={R} L={L}: {ms * 1e3:.1f} us per apply (CTA 0 total {t[:7].sum() / 1e3:.1f} us)")
    for i, nm in enumerate(NAMES):
        print(f"   {nm:12s} {t[i] / 1e3:9.1f} us")

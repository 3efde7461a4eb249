"""Per-phase timing of the split TensorSketch kernel (CTA 0, debug hook
ids_debug_ts_split_timing) at C4/C5.  Usage: python tools/exp_ts_split_phases.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native

lib = _native.load()
lib.ids_debug_ts_split_timing.argtypes = [ctypes.c_void_p]
NAMES = ["scatter loads", "rank passes", "fft passes 1-2", "last+untangle", "spectrum/pack",
         "inverse passes", "exchange+out", "load wait", "first rows", "barrier 1"]
for name, N, I, R, L in (("C4", 3, 1000, 1000, 4096), ("C5", 4, 10000, 2000, 16384)):
    g = torch.Generator(device="cuda").manual_seed(5)
    fac = [torch.randn(R, I, generator=g, device="cuda", dtype=torch.float64).t() for _ in range(N)]
    w = torch.rand(R, generator=g, device="cuda", dtype=torch.float64) + 0.5
    op = ids.TensorSketchOp([I] * N, L, seed=1)
    for _ in range(3):
        op.apply_device(fac, w, norms=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        op.apply_device(fac, w, norms=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    buf = torch.zeros(16, dtype=torch.int64, device="cuda")
    lib.ids_debug_ts_split_timing(buf.data_ptr())
    op.apply_device(fac, w, norms=True)
    torch.cuda.synchronize()
    lib.ids_debug_ts_split_timing(None)
    t = buf.cpu().numpy()
    print(f"{name}: N={N} I={I} R={R} L={L}: {ms * 1e3:.1f} us per apply (CTA 0 total {t[:10].sum() / 1e3:.1f} us)")
    for i, nm in enumerate(NAMES):
        print(f"   {nm:16s} {t[i] / 1e3:9.1f} us")

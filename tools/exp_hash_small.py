"""Small-band knobs of the chain: lowest speculative band (kmin) and the band
size below which tails use the one-draw-per-lane walk."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native

lib = _native.load()
lib.ids_debug_fy_small.argtypes = [ctypes.c_int, ctypes.c_int64]


def timeit(I, L, n=10):
    for _ in range(2):
        ids.CountSketchOp(I, L, seed=1, surjective=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        ids.CountSketchOp(I, L, seed=10 + i, surjective=True)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


base = ids.CountSketchOp(10**6, 100, seed=3, surjective=True).bucket.copy()
for kmin in (12, 11, 10, 9):
    for wb in (16384, 8192, 4096, 1024, 1):
        lib.ids_debug_fy_small(kmin, wb)
        same = np.array_equal(ids.CountSketchOp(10**6, 100, seed=3, surjective=True).bucket, base)
        print(f"kmin={kmin} walk1_below={wb}: 1e7 {timeit(10**7, 200):.3f} ms, 1e6 {timeit(10**6, 100):.3f} ms, same={same}", flush=True)
lib.ids_debug_fy_small(12, 16384)

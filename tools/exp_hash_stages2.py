"""Sweep of the staged draw's knobs at I = 1e7 / 1e6: CTAs per SM of the side
applications, bands per stage."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native

lib = _native.load()
raw = ctypes.CDLL(lib._name) if hasattr(lib, "_name") else lib
raw.ids_debug_fy_side.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]


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


for I, L in ((10_000_000, 200), (1_000_000, 100)):
    lib.ids_set_hash_stages(1, 1 << 17)
    print(f"I={I} unstaged: {timeit(I, L):.3f} ms", flush=True)
    for stages in (2, 3):
        lib.ids_set_hash_stages(stages, 1 << 17)
        for per_sm in (1, 2, 4, 16):
            for b0, b1 in ((1, 1), (1, 2), (2, 2), (2, 3), (3, 2), (3, 3)):
                if stages == 2 and b1 != 2:
                    continue
                raw.ids_debug_fy_side(per_sm, b0, b1)
                print(f"I={I} stages={stages} side/SM={per_sm} bands=({b0},{b1}): {timeit(I, L):.3f} ms", flush=True)

"""Chain knobs after the stitch / re-run changes: CTAs per SM of the chain
kernel, chunk-length rule, second-epoch threshold; unstaged and staged draws
at I = 1e7 and 1e6 (time per draw from kernel timelines is in
prof_hash_timeline.py; here back-to-back draws, events)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native

lib = _native.load()
lib.ids_debug_fy_per_sm.argtypes = [ctypes.c_int]
lib.ids_debug_phaseb_chunks.argtypes = [ctypes.c_double, ctypes.c_int64]
lib.ids_debug_fy_e2_min.argtypes = [ctypes.c_double]


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


for stages in (1, 3):
    lib.ids_set_hash_stages(stages, 1 << 21)
    for per_sm in (2, 3, 4, 6, 8):
        lib.ids_debug_fy_per_sm(per_sm)
        print(f"stages={stages} chain CTAs/SM={per_sm}: 1e7 {timeit(10**7, 200):.3f} ms, 1e6 {timeit(10**6, 100):.3f} ms", flush=True)
    lib.ids_debug_fy_per_sm(2)
    for mul, tmax in ((1.6, 4096), (1.6, 8192), (0.8, 4096), (0.8, 2048), (3.2, 4096), (1.15, 4096)):
        lib.ids_debug_phaseb_chunks(mul, tmax)
        print(f"stages={stages} tmul={mul} tmax={tmax}: 1e7 {timeit(10**7, 200):.3f} ms, 1e6 {timeit(10**6, 100):.3f} ms", flush=True)
    lib.ids_debug_phaseb_chunks(0, 0)
    for th in (0.0, 2.0**14, 2.0**16, 2.0**18, 2.0**20, 1e30):
        lib.ids_debug_fy_e2_min(th)
        print(f"stages={stages} e2 min draws={th:.3g}: 1e7 {timeit(10**7, 200):.3f} ms, 1e6 {timeit(10**6, 100):.3f} ms", flush=True)
    lib.ids_debug_fy_e2_min(65536.0)

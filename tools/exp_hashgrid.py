"""Phase-B grid scaling and concurrent hash streams (I = 1e6, L = 100)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native

lib = _native.load()
lib.ids_set_hash_grid_cap.argtypes = [ctypes.c_int]
I, L = 10**6, 100


def one(seed):
    return ids.CountSketchOp(I, L, seed=seed, surjective=True)._bucket_index()


for cap in (0, 148, 74, 37, 18):
    lib.ids_set_hash_grid_cap(cap)
    one(1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(5):
        one(10 + s)
    e1.record()
    torch.cuda.synchronize()
    print(f"cap {cap:4d}: {e0.elapsed_time(e1) / 5 * 1e3:8.1f} us per hash+index")
for K, cap in ((10, 29), (10, 18), (5, 59), (4, 74)):
    lib.ids_set_hash_grid_cap(cap)
    streams = [torch.cuda.Stream() for _ in range(K)]
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        outs = []
        for k, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                outs.append(one(100 + k))
        for s in streams:
            e1.wait_stream(s) if hasattr(e1, "wait_stream") else torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    print(f"K={K} streams cap {cap}: {e0.elapsed_time(e1) * 1e3:8.1f} us total, "
          f"{e0.elapsed_time(e1) / K * 1e3:8.1f} us per hash")
lib.ids_set_hash_grid_cap(0)

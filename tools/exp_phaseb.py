import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native
lib = _native.load()
buf = torch.zeros(512, dtype=torch.int64, device="cuda")
lib.ids_debug_phaseb_timing.argtypes = [ctypes.c_void_p]
cap = int(os.environ.get("CAP", "0"))
lib.ids_set_hash_grid_cap(cap)
for I in (10**6, 10**7):
    ids.CountSketchOp(I, 100, seed=1, surjective=True)._bucket_index()
    buf.zero_()
    lib.ids_debug_phaseb_timing(buf.data_ptr())
    ids.CountSketchOp(I, 100, seed=2, surjective=True)._bucket_index()
    torch.cuda.synchronize()
    lib.ids_debug_phaseb_timing(None)
    t = buf.cpu().numpy()
    tags, ts = t[0::2], t[1::2]
    n = int(np.argmax(tags == -1)) if (tags == -1).any() else len(tags)
    t0 = ts[0]
    prev = t0
    print(f"I={I}")
    for k in range(n):
        print(f"  tag {tags[k]:5d}  t={(ts[k]-t0)/1e3:9.1f} us  (+{(ts[k]-prev)/1e3:7.1f})")
        prev = ts[k]

# whole hash (draws + Fisher-Yates + signs + bucket index), device time
for I, L in ((10**6, 100), (10**7, 200)):
    ts = []
    for s in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ids.CountSketchOp(I, L, seed=10 + s, surjective=True)._bucket_index()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"hash I={I}: median {sorted(ts[1:])[2] * 1e3:.0f} us", flush=True)

# chunk-length rule sweep (ids_debug_phaseb_chunks)
lib.ids_debug_phaseb_chunks.argtypes = [ctypes.c_double, ctypes.c_int64]
for mul, tmax in ((2.3, 4096), (1.15, 4096), (1.15, 8192), (0.8, 4096), (0.575, 4096), (1.6, 4096), (1.6, 8192)):
    lib.ids_debug_phaseb_chunks(mul, tmax)
    out = []
    for I, L in ((10**6, 100), (10**7, 200)):
        ts = []
        for s in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            op = ids.CountSketchOp(I, L, seed=40 + s, surjective=True)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out.append(f"I={I}: {sorted(ts)[2] * 1e3:.0f} us")
    print(f"mul {mul} tmax {tmax}: " + ", ".join(out), flush=True)
lib.ids_debug_phaseb_chunks(0, 0)

# cooperative-groups grid.sync vs the nanosleep barrier (ids_debug_fy_custom_bar)
lib.ids_debug_fy_custom_bar.argtypes = [ctypes.c_int]
for cb in (0, 1, 0, 1):
    lib.ids_debug_fy_custom_bar(cb)
    out = []
    for I, L in ((10**6, 100), (10**7, 200)):
        ts = []
        for s in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            op = ids.CountSketchOp(I, L, seed=70 + s, surjective=True)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ref = oracle_ok = None
        out.append(f"I={I}: {sorted(ts)[2] * 1e3:.0f} us")
    print(f"custom barrier {cb}: " + ", ".join(out), flush=True)
lib.ids_debug_fy_custom_bar(1)

# second-epoch threshold (ids_debug_fy_e2_min)
lib.ids_debug_fy_e2_min.argtypes = [ctypes.c_double]
for th in (0.0, 2.0**14, 2.0**16, 2.0**18, 2.0**20, 1e30, 0.0):
    lib.ids_debug_fy_e2_min(th)
    out = []
    for I, L in ((10**6, 100), (10**7, 200)):
        ts = []
        for s in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            op = ids.CountSketchOp(I, L, seed=110 + s, surjective=True)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out.append(f"I={I}: {sorted(ts)[2] * 1e3:.0f} us")
    print(f"e2 min draws {th:.3g}: " + ", ".join(out), flush=True)
lib.ids_debug_fy_e2_min(65536.0)

"""Per-band stage timestamps of the (unstaged) phase-B chain kernel
(ids_debug_phaseb_timing) at I = 1e6 and 1e7."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native
lib = _native.load()
buf = torch.zeros(512, dtype=torch.int64, device="cuda")
lib.ids_debug_phaseb_timing.argtypes = [ctypes.c_void_p]
for I in (10**6, 10**7):
    ids.CountSketchOp(I, 100, seed=1, surjective=True)
    buf.zero_()
    lib.ids_debug_phaseb_timing(buf.data_ptr())
    ids.CountSketchOp(I, 100, seed=2, surjective=True)
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

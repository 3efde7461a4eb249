"""Kernel timeline (torch profiler / CUPTI) of one surjective hash draw at
I = 1e7 for 1 and 3 stages: start offset, duration of every kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native

lib = _native.load()
I, L = int(os.environ.get("I", 10_000_000)), 200
for stages in (1, 3):
    lib.ids_set_hash_stages(stages, 1 << 17)
    for _ in range(2):
        ids.CountSketchOp(I, L, seed=1, surjective=True)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        ids.CountSketchOp(I, L, seed=2, surjective=True)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start
    print(f"--- stages={stages}")
    for e in evs:
        print(f"{(e.time_range.start - t0):9.1f} us  +{e.time_range.elapsed_us():8.1f}  {e.name[:60]}")
    print(f"total {(max(e.time_range.end for e in evs) - t0):.1f} us", flush=True)

"""Kernel timeline of single C4 tensor-ID calls on device-resident factors:
every kernel / copy with its start, duration and the idle gaps."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
from paper_1901_10559_b200 import generators as G
from paper_1901_10559_b200.distributed import tensorsketch_id_sharded

torch.cuda.set_device(0)
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = G.CONFIGS[name]
w, facs = G.cp_config(name)
wh = w.cpu().numpy()


class X:
    factors = facs
    weights = w
    mode_dims = tuple([cfg["dim"]] * cfg["modes"])


def call(s):
    return tensorsketch_id_sharded(X, 0, cfg["terms"], wh, cfg["k"], cfg["L"], seed=s)


for s in range(3):
    call(s)
torch.cuda.synchronize()
t0 = time.perf_counter()
for s in range(20):
    call(100 + s)
print("wall per call %.3f ms" % ((time.perf_counter() - t0) / 20 * 1e3))
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    call(7)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
end = t0
busy = 0.0
for e in evs:
    s, d = e.time_range.start, e.time_range.elapsed_us()
    gap = s - end
    busy += d
    print(f"  {s - t0:8.1f} +{d:7.1f} gap {gap:6.1f}  {e.name[:70]}")
    end = max(end, s + d)
print("span", end - t0, "busy", busy, "kernels", len(evs))

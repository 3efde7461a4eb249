"""Kernel timeline (torch profiler) of one countsketch_id call on the device
operand of C2 or C3: start offset, duration and gap before every kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import generators as G
from paper_1901_10559_b200._inputs import dense_operand

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = G.CONFIGS[wl]
a = dense_operand(G.dense_config(wl)) if cfg["kind"] == "dense" else G.csr_config(wl)
for s in range(3):
    ids.countsketch_id(a, cfg["k"], cfg["L"], seed=s)
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
ids.countsketch_id(a, cfg["k"], cfg["L"], seed=7)
print(f"wall {1e3 * (time.perf_counter() - t0):.3f} ms (no profiler)")
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    ids.countsketch_id(a, cfg["k"], cfg["L"], seed=9)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
end = t0
for e in evs:
    gap = e.time_range.start - end
    print(f"{(e.time_range.start - t0):9.1f} us  +{e.time_range.elapsed_us():8.1f}  gap {gap:7.1f}  {e.name[:70]}")
    end = max(end, e.time_range.end)
print(f"total {(end - t0):.1f} us")

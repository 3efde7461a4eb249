"""Kernel timeline of queued C4/C5 tensor-ID trials replayed from the
captured graph (TensorIdGraph.trials): every kernel with start, duration and
idle gaps.  Usage: python tools/exp_timeline_graph.py C5"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_1901_10559_b200 import generators as G
from paper_1901_10559_b200.cp_tensor import TensorIdGraph

torch.cuda.set_device(0)
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = G.CONFIGS[name]
w, facs = G.cp_config(name)
gr = TensorIdGraph(facs, w, cfg["k"], cfg["L"], host_weights=w.cpu().numpy())
gr.trials(range(3))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
gr.trials(range(10, 30))
e1.record()
torch.cuda.synchronize()
print("per trial %.3f ms" % (e0.elapsed_time(e1) / 20))
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    gr.trials(range(100, 102))
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
end = t0
for e in evs:
    s, d = e.time_range.start, e.time_range.elapsed_us()
    print(f"  {s - t0:8.1f} +{d:7.1f} gap {s - end:6.1f}  {e.name[:70]}")
    end = max(end, s + d)
print("span", end - t0)

"""Kernel timeline (torch.profiler / CUPTI) of queued C3 trials: prints the
kernels longer than 50 us and every idle gap above 20 us."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_1901_10559_b200 import generators as G
from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials

torch.cuda.set_device(0)
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = G.CONFIGS[name]
from paper_1901_10559_b200._inputs import dense_operand
a = G.csr_config(name) if cfg["kind"] == "csr" else dense_operand(G.dense_config(name))
rows, k, L = cfg["rows"], cfg["k"], cfg["L"]
cap = int(sys.argv[3]) if len(sys.argv) > 3 else 0
countsketch_id_sharded_trials(a, 0, rows, k, L, seeds=range(6), depth=depth, grid_cap=cap)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    countsketch_id_sharded_trials(a, 0, rows, k, L, seeds=range(100, 106), depth=depth, grid_cap=cap)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
end = t0
for e in evs:
    s, d = e.time_range.start, e.time_range.elapsed_us()
    if s - end > 20:
        print(f"  GAP {s - end:8.1f} before {e.name[:60]}")
    if d > 50 or "--all" in sys.argv:
        print(f"  {s - t0:9.1f} +{d:8.1f}  {e.name[:70]}")
    end = max(end, s + d)
print("total", end - t0)
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and "cuda" in e.name.lower() and e.cpu_time_total > 200]
for e in cpu[:30]:
    print("CPU", e.name, e.cpu_time_total)

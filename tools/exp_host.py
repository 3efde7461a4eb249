"""Host-side cost of one tensor ID step (C4 shape) under cProfile, and the
GPU-idle gap: wall time vs device time."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200.matrix_id import device_matrix_id

N, I, R, K, L = 3, 1000, 1000, 10, 4096
g = torch.Generator(device="cuda").manual_seed(4)
facs = [torch.randn(R, I, generator=g, device="cuda", dtype=torch.float64).t() for _ in range(N)]
w = torch.rand(R, generator=g, device="cuda", dtype=torch.float64) + 0.5


def step(s):
    y = ids.TensorSketchOp([I] * N, L, seed=s).apply_device(facs, w)
    return device_matrix_id(y, L, R, K).to_host("tensorsketch")


for s in range(5):
    step(s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for s in range(20):
    step(100 + s)
e1.record()
torch.cuda.synchronize()
print(f"wall {1e3 * (time.perf_counter() - t0) / 20:.3f} ms/step, device {e0.elapsed_time(e1) / 20:.3f} ms/step")
pr = cProfile.Profile()
pr.enable()
for s in range(20):
    step(200 + s)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)

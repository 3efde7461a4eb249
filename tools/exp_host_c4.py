"""Host-side cost of one C4 tensorsketch_id step (Python + ctypes + launches),
against its device time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200.matrix_id import device_matrix_id

N, In, R, L, K = 3, 1000, 1000, 4096, 10
g = torch.Generator(device="cuda").manual_seed(4)
facs = [torch.randn(R, In, generator=g, device="cuda", dtype=torch.float64).t() for _ in range(N)]
w = torch.rand(R, generator=g, device="cuda", dtype=torch.float64) + 0.5
for s in range(5):
    y = ids.TensorSketchOp([In] * N, L, seed=s).apply_device(facs, w)
    device_matrix_id(y, L, R, K).to_host("tensorsketch")
torch.cuda.synchronize()
for s in range(3):
    t0 = time.perf_counter()
    op = ids.TensorSketchOp([In] * N, L, seed=100 + s)
    t1 = time.perf_counter()
    y = op.apply_device(facs, w)
    t2 = time.perf_counter()
    d = device_matrix_id(y, L, R, K)
    t3 = time.perf_counter()
    d.to_host("tensorsketch")
    t4 = time.perf_counter()
    print(f"host: op {1e3*(t1-t0):.3f} ms, apply {1e3*(t2-t1):.3f}, id launch {1e3*(t3-t2):.3f}, to_host(sync) {1e3*(t4-t3):.3f}, total {1e3*(t4-t0):.3f}")

"""Column-distributed CPQR (device-driven, fused launches) on one GPU: a full C5-shaped
sketch and a 1/8 column shard (what each of 8 ranks runs, minus the two
collectives per step), host enqueue time vs device time, against the
single-GPU cpqr_kernel."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_10559_b200.distributed import DeviceCpqrShard, _dcpqr_device
from paper_1901_10559_b200.matrix_id import device_matrix_id

torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(1)
m, n, k = 16384, 2000, 20
base = torch.randn(m, 20, generator=g, device="cuda", dtype=torch.float64)
idx = torch.randint(0, 20, (n,), generator=g, device="cuda")
y = (base[:, idx] + 1e-4 * torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)).t().contiguous()


def run(label, fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        fn()
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    print(f"{label}: device {e0.elapsed_time(e1) / reps:.3f} ms, host enqueue {(t1 - t0) / reps * 1e3:.3f} ms")


run("cpqr_kernel (2000 cols)", lambda: device_matrix_id(y, m, n, k))
run("dcpqr world 1 (2000 cols)", lambda: _dcpqr_device(DeviceCpqrShard(y, 0, k), [(0, n)], n, k, 1e-12, None))
ys = y[:250].contiguous()
run("dcpqr shard (250 cols)", lambda: _dcpqr_device(DeviceCpqrShard(ys, 0, k), [(0, 250)], 250, k, 1e-12, None))

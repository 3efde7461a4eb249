"""Trials throughput (C2 shape, 10 trials) for several hash-pipeline settings."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_10559_b200 import sketch
from paper_1901_10559_b200._inputs import dense_operand
from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials

I, R = 1_000_000, 2000
a = torch.randn(I, R, dtype=torch.float64, device="cuda")
op = dense_operand(a)
countsketch_id_sharded_trials(op, 0, I, 20, 100, seeds=list(range(12)))
for depth, cap in ((2, 16), (2, 8), (2, 4), (3, 8), (1, 8), (2, 16)):
    sketch.PIPELINE_DEPTH, sketch.PIPELINE_GRID_CAP = depth, cap
    countsketch_id_sharded_trials(op, 0, I, 20, 100, seeds=list(range(4)))
    torch.cuda.synchronize()
    best, allr = 1e9, []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        countsketch_id_sharded_trials(op, 0, I, 20, 100, seeds=list(range(100 + 20 * rep, 120 + 20 * rep)))
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 20)
        allr.append(round(e0.elapsed_time(e1) / 20 * 1e3))
    print(f"depth {depth} cap {cap:3d}: {best * 1e3:7.0f} us per trial {allr}", flush=True)

# main-stream work alone: one pre-drawn operator reused for every trial
from paper_1901_10559_b200.matrix_id import device_matrix_id
import paper_1901_10559_b200 as ids
fixed = ids.CountSketchOp(I, 100, seed=7, surjective=True)
fixed.bucket_index()
def no_hash_trials(n):
    outs = []
    for _ in range(n):
        y = torch.empty((R, 100), dtype=torch.float64, device="cuda")
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        fixed.sketch_into(op, y, flags=1, nonfinite=flag)
        outs.append(device_matrix_id(y, 100, R, 20).packed())
    return torch.stack(outs).cpu()
no_hash_trials(3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
no_hash_trials(10)
e1.record()
torch.cuda.synchronize()
print(f"no hash (fixed operator): {e0.elapsed_time(e1) / 20 * 1e3:7.0f} us per trial", flush=True)

# sketch alone, and CPQR moved to a high-priority side stream
def sketch_only(n):
    y = torch.empty((R, 100), dtype=torch.float64, device="cuda")
    for _ in range(n):
        fixed.sketch_into(op, y, flags=1)
    return y

side = torch.cuda.Stream(priority=-1)
def side_cpqr_trials(n):
    outs = []
    main = torch.cuda.current_stream()
    for _ in range(n):
        y = torch.empty((R, 100), dtype=torch.float64, device="cuda")
        fixed.sketch_into(op, y, flags=1)
        ev = torch.cuda.Event()
        ev.record()
        with torch.cuda.stream(side):
            side.wait_event(ev)
            outs.append(device_matrix_id(y, 100, R, 20).packed())
            y.record_stream(side)
    main.wait_stream(side)
    return torch.stack(outs).cpu()

for name, fn in (("sketch only", sketch_only), ("cpqr on side stream", side_cpqr_trials)):
    fn(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(10)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 20 * 1e3:7.0f} us per trial", flush=True)

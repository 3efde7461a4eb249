"""Repeated timings of the C2 trials batch in one process (first-run effects)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_10559_b200._inputs import dense_operand
from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials

I, R = 1_000_000, 2000
a = torch.randn(I, R, dtype=torch.float64, device="cuda")
op = dense_operand(a)
countsketch_id_sharded_trials(op, 0, I, 20, 100, seeds=list(range(10)))
torch.cuda.synchronize()
for rep in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    countsketch_id_sharded_trials(op, 0, I, 20, 100, seeds=list(range(100 + 10 * rep, 110 + 10 * rep)))
    e1.record()
    torch.cuda.synchronize()
    print(f"rep {rep}: {e0.elapsed_time(e1) / 10 * 1e3:7.0f} us per trial, wall {(time.perf_counter() - t0) * 1e3:7.1f} ms",
          flush=True)

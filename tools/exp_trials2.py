"""Timing of concurrent hash draws (draw_operators) and the trials API."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200.sketch import draw_operators
from paper_1901_10559_b200._inputs import dense_operand
from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials

I, L = 10**6, 100


def timed(fn, label):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{label}: gpu {e0.elapsed_time(e1):8.2f} ms  wall {1e3 * (time.perf_counter() - t0):8.2f} ms",
          flush=True)


for rep in range(3):
    timed(lambda: draw_operators(I, L, list(range(10 * rep, 10 * rep + 10)), True), f"draw10 rep{rep}")
for rep in range(2):
    timed(lambda: [ids.CountSketchOp(I, L, seed=s, surjective=True)._bucket_index() for s in range(10)],
          f"seq10 rep{rep}")
a = torch.randn(200_000, 2000, dtype=torch.float64, device="cuda")
op = dense_operand(a)
for rep in range(3):
    timed(lambda: countsketch_id_sharded_trials(op, 0, 200_000, 20, 100, seeds=list(range(10))),
          f"trials10 (200k rows) rep{rep}")

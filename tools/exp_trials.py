"""Experiment: per-trial timing variants for the C2 countsketch_id loop."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200._inputs import dense_operand
from paper_1901_10559_b200.distributed import countsketch_id_sharded, countsketch_id_sharded_trials

a = torch.randn(1_000_000, 2000, dtype=torch.float64, device="cuda")
op = dense_operand(a)
N = 10

def timeit(fn, label):
    fn(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(1)
    e1.record()
    torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1)/N:.3f} ms/trial (wall {1e3*(time.perf_counter()-t0)/N:.3f})", flush=True)

timeit(lambda b: [countsketch_id_sharded(op, 0, 10**6, 20, 100, seed=b*100+s) for s in range(N)], "plain per-call")
timeit(lambda b: countsketch_id_sharded_trials(op, 0, 10**6, 20, 100, seeds=[b*100+s for s in range(N)]), "trials")
def hash_only(b):
    for s in range(N):
        ids.CountSketchOp(10**6, 100, seed=b*100+s, surjective=True)._bucket_index()
timeit(hash_only, "hash+index only")
def hash_sync(b):
    for s in range(N):
        ids.CountSketchOp(10**6, 100, seed=b*100+s, surjective=True)._bucket_index()
        torch.cuda.synchronize()
timeit(hash_sync, "hash+index only (sync each)")
y = torch.empty((2000, 100), dtype=torch.float64, device="cuda")
o2 = ids.CountSketchOp(10**6, 100, seed=1, surjective=True)
timeit(lambda b: [o2.sketch_into(op, y, flags=1) for s in range(N)], "sketch only")

import sys, os
sys.path.insert(0, "/root/repo")
import torch
from paper_1901_10559_b200 import generators as G
from paper_1901_10559_b200._inputs import dense_operand
from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials
torch.cuda.set_device(0)
cfg = G.CONFIGS["C2"]
a = dense_operand(G.dense_config("C2"))
rows, k, L = cfg["rows"], cfg["k"], cfg["L"]
print("priority range", torch.cuda.Stream.priority_range())
def timeit(stream, tag):
    with torch.cuda.stream(stream):
        countsketch_id_sharded_trials(a, 0, rows, k, L, seeds=range(20))
        torch.cuda.synchronize()
        ts = []
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            countsketch_id_sharded_trials(a, 0, rows, k, L, seeds=range(1000 + 20 * rep, 1020 + 20 * rep))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 20)
    print(tag, ["%.3f" % t for t in ts])
lo, hi = torch.cuda.Stream.priority_range()
timeit(torch.cuda.current_stream(), "default prio")
for p in sorted(set([hi, hi + 1 if hi + 1 <= lo else hi, lo])):
    timeit(torch.cuda.Stream(priority=p), f"sketch prio {p}")

"""C3 trials (K = 20 seeds of countsketch_id on the device CSR): time per
trial with the hash draws under the sketches (pipelined) or batched ahead
of them (several concurrent capped draws, then the sketches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_10559_b200 import generators as G
from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials

op = G.csr_config("C3")
I = op.rows
countsketch_id_sharded_trials(op, 0, I, 20, 200, seeds=list(range(3)))
settings = [("pipelined depth 2 full grid", dict(batched=False, depth=2, grid_cap=0)),
            ("batched 4 x 74 CTAs", dict()),
            ("batched 4 x 37 CTAs", dict(grid_cap=37)),
            ("batched 8 x 37 CTAs", dict(streams=8, grid_cap=37)),
            ("batched 8 x 18 CTAs", dict(streams=8, grid_cap=18)),
            ("batched 4 x 74, batch 20", dict(batch=20)),
            ("batched 4 x 74, batch 8", dict(batch=8))]
for name, kw in settings:
    countsketch_id_sharded_trials(op, 0, I, 20, 200, seeds=list(range(4)), **dict(kw))
    torch.cuda.synchronize()
    res = []
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        countsketch_id_sharded_trials(op, 0, I, 20, 200, seeds=list(range(100 + 20 * rep, 120 + 20 * rep)),
                                      **dict(kw))
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 20)
    print(f"{name:28s}: {min(res):.3f} ms per trial {[round(r, 3) for r in res]}", flush=True)

"""C3 trials (K = 20 seeds of countsketch_id on the device CSR): time per
trial for several background hash-draw settings (look-ahead depth, phase-B
CTAs per draw; 0 = full grid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_10559_b200 import generators as G
from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials

op = G.csr_config("C3")
I = op.rows
countsketch_id_sharded_trials(op, 0, I, 20, 200, seeds=list(range(3)))
settings = [(2, 0), (3, 148), (4, 148), (3, 296), (4, 74), (6, 148), (8, 74), (2, 0)]
for depth, cap in settings:
    kw = dict(depth=depth, grid_cap=cap)
    countsketch_id_sharded_trials(op, 0, I, 20, 200, seeds=list(range(4)), **kw)
    torch.cuda.synchronize()
    res = []
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        countsketch_id_sharded_trials(op, 0, I, 20, 200, seeds=list(range(100 + 20 * rep, 120 + 20 * rep)),
                                      **kw)
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 20)
    print(f"depth {depth} cap {cap:3d}: {min(res):.3f} ms per trial {[round(r, 3) for r in res]}", flush=True)

"""C2 trials (20 seeds): time per trial against the look-ahead depth and the
phase-B grid cap of the background hash draws."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_10559_b200 import generators as G
from paper_1901_10559_b200._inputs import dense_operand
from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials

a = dense_operand(G.dense_config("C2"))
I = a.rows
countsketch_id_sharded_trials(a, 0, I, 20, 100, seeds=list(range(3)))
for depth, cap in ((2, 16), (2, 8), (2, 32), (2, 74), (1, 16), (1, 74), (1, 148), (3, 16), (3, 8), (2, 4), (2, 16)):
    res = []
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        countsketch_id_sharded_trials(a, 0, I, 20, 100, seeds=list(range(100 + 20 * rep, 120 + 20 * rep)),
                                      depth=depth, grid_cap=cap)
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / 20)
    print(f"depth {depth} cap {cap:3d}: {min(res):.3f} ms per trial {[round(r, 3) for r in res]}", flush=True)

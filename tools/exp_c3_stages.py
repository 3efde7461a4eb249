"""C3 with the staged hash draw (ids_set_hash_stages 1 vs 3): single-call
countsketch_id and 20 trials (batched draws, several settings)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native, generators as G
from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials

lib = _native.load()
op = G.csr_config("C3")
I = op.rows
for stages in (1, 3, 1, 3):
    lib.ids_set_hash_stages(stages, 0)
    for _ in range(2):
        ids.countsketch_id(op, 20, 200, seed=1)
    ts = []
    for s in range(7):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ids.countsketch_id(op, 20, 200, seed=10 + s)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"stages={stages} single call: median {sorted(ts)[3]:.3f} ms {[round(t, 2) for t in ts]}", flush=True)
    for name, kw in (("batched 4 x 74", dict()), ("batched 4 x 148", dict(grid_cap=148)),
                     ("batched 2 x 148", dict(streams=2, grid_cap=148)),
                     ("batched 8 x 37", dict(streams=8, grid_cap=37))):
        countsketch_id_sharded_trials(op, 0, I, 20, 200, seeds=list(range(4)), **dict(kw))
        res = []
        for rep in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            countsketch_id_sharded_trials(op, 0, I, 20, 200,
                                          seeds=list(range(100 + 20 * rep, 120 + 20 * rep)), **dict(kw))
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) / 20)
        print(f"stages={stages} trials {name:16s}: {min(res):.3f} ms per trial {[round(r, 3) for r in res]}", flush=True)

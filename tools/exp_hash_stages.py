"""Staged surjective hash draw (ids_set_hash_stages): buckets / signs against
the unstaged draw at several sizes, and the time per draw for 1 / 2 / 3
stages at I = 1e6 (C2) and I = 1e7 (C3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native

lib = _native.load()


def draw(I, L, seed, stages):
    lib.ids_set_hash_stages(stages, 1 << 17)
    op = ids.CountSketchOp(I, L, seed=seed, surjective=True)
    torch.cuda.synchronize()
    return op


for I, L in ((131072 + 5, 40), (300_000, 7), (1 << 20, 100), (1_000_000, 100), ((1 << 21) + 1, 3),
             (4_194_303, 64), (10_000_000, 200)):
    for seed in (0, 5):
        base = draw(I, L, seed, 1)
        for stages in (2, 3):
            op = draw(I, L, seed, stages)
            same = np.array_equal(op.bucket, base.bucket) and np.array_equal(op.sign, base.sign)
            print(f"I={I} L={L} seed={seed} stages={stages}: {'same' if same else 'DIFFERENT'}", flush=True)

for I, L in ((1_000_000, 100), (10_000_000, 200)):
    for stages in (1, 2, 3):
        lib.ids_set_hash_stages(stages, 1 << 17)
        for _ in range(3):
            ids.CountSketchOp(I, L, seed=1, surjective=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 10
        e0.record()
        for i in range(n):
            ids.CountSketchOp(I, L, seed=10 + i, surjective=True)
        e1.record()
        torch.cuda.synchronize()
        print(f"I={I} stages={stages}: {e0.elapsed_time(e1) / n:.3f} ms per draw (back to back)", flush=True)
lib.ids_set_hash_stages(3, 1 << 19)

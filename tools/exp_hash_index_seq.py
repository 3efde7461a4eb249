"""Back-to-back CountSketchOp(...).bucket_index() at I = 1e7 (what bench.py's
hash_and_index phase times): per-call event times, staged vs unstaged."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native

lib = _native.load()
I, L = 10**7, 200
for stages in (1, 3, 1, 3):
    lib.ids_set_hash_stages(stages, 0)
    for with_index in (False, True):
        ts = []
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(9)]
        torch.cuda.synchronize()
        evs[0].record()
        for i in range(8):
            op = ids.CountSketchOp(I, L, seed=100 + i, surjective=True)
            if with_index:
                op.bucket_index()
            evs[i + 1].record()
        torch.cuda.synchronize()
        ts = [round(evs[i].elapsed_time(evs[i + 1]), 2) for i in range(8)]
        print(f"stages={stages} index={with_index}: {ts}", flush=True)

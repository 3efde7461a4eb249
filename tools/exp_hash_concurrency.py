"""Throughput of surjective CountSketch hash draws (I = 1e7, L = 200, the
C3 operator) run 2 / 4 / 8 at a time on separate streams, with the phase-B
grid capped at 148 / 74 / 37 / 18 CTAs per draw."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native

lib = _native.load()
I, L = 10_000_000, 200
streams = [torch.cuda.Stream() for _ in range(8)]
ids.CountSketchOp(I, L, seed=1, surjective=True)
torch.cuda.synchronize()
for cap in (148, 74, 37, 18):
    lib.ids_set_hash_grid_cap(cap)
    for conc in (2, 4, 8):
        n = 16
        ops = []
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        main = torch.cuda.current_stream()
        for i in range(n):
            st = streams[i % conc]
            st.wait_stream(main) if i < conc else None
            with torch.cuda.stream(st):
                ops.append(ids.CountSketchOp(I, L, seed=100 + i, surjective=True))
        for st in streams[:conc]:
            main.wait_stream(st)
        e1.record()
        torch.cuda.synchronize()
        print(f"cap {cap:3d} concurrent {conc}: {e0.elapsed_time(e1) / n:.3f} ms per draw", flush=True)
    lib.ids_set_hash_grid_cap(0)

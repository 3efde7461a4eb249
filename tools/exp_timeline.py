"""Event timeline of the trials pipeline (C2 shape): per trial, when its hash
draw, sketch and ID start and end (CUDA events on their own streams, ms from
the first event).  usage: python tools/exp_timeline.py [depth] [cap]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import sketch
from paper_1901_10559_b200._inputs import dense_operand
from paper_1901_10559_b200._native import load
from paper_1901_10559_b200.matrix_id import device_matrix_id

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 16
I, R, L, K = 1_000_000, 2000, 100, 20
a = torch.randn(I, R, dtype=torch.float64, device="cuda")
op_in = dense_operand(a)
lib = load()
dev = torch.device("cuda", 0)
sides = [torch.cuda.Stream() for _ in range(depth)]
idst = sketch.id_stream()
main = torch.cuda.current_stream()


def ev(st=None):
    e = torch.cuda.Event(enable_timing=True)
    e.record(st) if st is not None else e.record()
    return e


def run(seeds, log):
    t0 = ev()
    first = ids.CountSketchOp(I, L, seed=seeds[0], surjective=True)
    first._bucket_index()
    pending = [(first, None, None, None)]
    nxt = 1
    outs = []
    for i in range(len(seeds)):
        while nxt < len(seeds) and nxt <= i + depth:
            lib.ids_set_hash_grid_cap(cap)
            st = sides[nxt % len(sides)]
            with torch.cuda.stream(st):
                h0 = ev(st)
                op = ids.CountSketchOp(I, L, seed=seeds[nxt], surjective=True)
                op._bucket_index()
                h1 = ev(st)
            lib.ids_set_hash_grid_cap(0)
            pending.append((op, h1, h0, h1))
            nxt += 1
        op, e, h0, h1 = pending.pop(0)
        if e is not None:
            main.wait_event(e)
        s0 = ev()
        y = torch.empty((R, L), dtype=torch.float64, device="cuda")
        op.sketch_into(op_in, y, flags=1)
        s1 = ev()
        idst.wait_stream(main)
        with torch.cuda.stream(idst):
            c0 = ev(idst)
            outs.append(device_matrix_id(y, L, R, K).packed())
            c1 = ev(idst)
        y.record_stream(idst)
        log.append((h0, h1, s0, s1, c0, c1))
    main.wait_stream(idst)
    torch.stack(outs).cpu()
    return t0


run(list(range(6)), [])
torch.cuda.synchronize()
log = []
t0 = run(list(range(100, 110)), log)
torch.cuda.synchronize()
f = lambda e: t0.elapsed_time(e) if e is not None else float("nan")
print(f"depth {depth} cap {cap}")
print(" trial   hash[start,end]      sketch[start,end]    id[start,end]")
for i, (h0, h1, s0, s1, c0, c1) in enumerate(log):
    print(f" {i:3d}  {f(h0):7.3f} {f(h1):7.3f}   {f(s0):7.3f} {f(s1):7.3f}   {f(c0):7.3f} {f(c1):7.3f}")

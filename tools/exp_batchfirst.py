"""Trials with all hash draws done first (side streams, concurrently), then
the sketches back to back with the IDs on the high-priority stream; against
the default depth-2 pipeline (C2 shape, 10 trials)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import sketch
from paper_1901_10559_b200._inputs import dense_operand
from paper_1901_10559_b200._native import load
from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials
from paper_1901_10559_b200.matrix_id import device_matrix_id

I, R, L, K = 1_000_000, 2000, 100, 20
a = torch.randn(I, R, dtype=torch.float64, device="cuda")
opnd = dense_operand(a)
lib = load()
main = torch.cuda.current_stream()
side = sketch.id_stream()


def batch_first(seeds, cap, nstreams):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    ops, evs = [], []
    for n, s in enumerate(seeds):
        lib.ids_set_hash_grid_cap(cap)
        with torch.cuda.stream(streams[n % nstreams]):
            op = ids.CountSketchOp(I, L, seed=s, surjective=True)
            op._bucket_index()
            ev = torch.cuda.Event()
            ev.record()
        lib.ids_set_hash_grid_cap(0)
        ops.append(op)
        evs.append(ev)
    for ev in evs:
        main.wait_event(ev)
    outs = []
    for op in ops:
        op.record_stream(main)
        y = torch.empty((R, L), dtype=torch.float64, device="cuda")
        op.sketch_into(opnd, y, flags=1)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            outs.append(device_matrix_id(y, L, R, K).packed())
        y.record_stream(side)
    main.wait_stream(side)
    return torch.stack(outs).cpu()


def timed(fn, label):
    fn(list(range(10)))
    torch.cuda.synchronize()
    res = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(list(range(100 + 10 * rep, 110 + 10 * rep)))
        e1.record()
        torch.cuda.synchronize()
        res.append(round(e0.elapsed_time(e1) / 10 * 1e3))
    print(f"{label}: {res} us per trial", flush=True)


timed(lambda s: countsketch_id_sharded_trials(opnd, 0, I, K, L, seeds=s), "pipeline depth 2")
for cap, ns in ((16, 10), (32, 5), (64, 3), (148, 1), (16, 4)):
    timed(lambda s, cap=cap, ns=ns: batch_first(s, cap, ns), f"batch first cap {cap} streams {ns}")

"""C3 trials split into their two phases: the 20 hash draws alone (batched
as batched_operators does), and the 20 sketches + IDs alone on pre-drawn
operators."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_10559_b200 import generators as G
from paper_1901_10559_b200._native import IDS_FLAG_ORDERED
from paper_1901_10559_b200.matrix_id import device_matrix_id
from paper_1901_10559_b200.sketch import batched_operators, id_stream

op_a = G.csr_config("C3")
I, R, L, k = op_a.rows, op_a.cols, 200, 20


def ev(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), out


def compute(ops, side_id=True):
    main, side = torch.cuda.current_stream(), id_stream()
    outs = []
    for op in ops:
        y = torch.empty((R, L), dtype=torch.float64, device="cuda")
        op.sketch_into(op_a, y, flags=IDS_FLAG_ORDERED)
        if side_id:
            side.wait_stream(main)
            with torch.cuda.stream(side):
                outs.append(device_matrix_id(y, L, R, k).packed())
            y.record_stream(side)
        else:
            outs.append(device_matrix_id(y, L, R, k).packed())
    main.wait_stream(side)
    return outs


ev(lambda: list(batched_operators(I, L, range(4), True, index=False)))
for rep in range(2):
    t, ops = ev(lambda: list(batched_operators(I, L, range(100 * rep, 100 * rep + 20), True, index=False)))
    print(f"draws only: {t / 20:.3f} ms per draw", flush=True)
    compute(ops[:3])
    t, _ = ev(lambda: compute(ops))
    print(f"sketch + ID (ID on side stream): {t / 20:.3f} ms per trial", flush=True)
    t, _ = ev(lambda: compute(ops, side_id=False))
    print(f"sketch + ID (serial): {t / 20:.3f} ms per trial", flush=True)
    t, _ = ev(lambda: [op.sketch_into(op_a, torch.empty((R, L), dtype=torch.float64, device='cuda'),
                                      flags=IDS_FLAG_ORDERED) for op in ops])
    print(f"sketch only: {t / 20:.3f} ms per trial", flush=True)

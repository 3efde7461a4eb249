"""Per-call wall time of tensorsketch_id from host factors (pinned, unit
columns) at C4/C5: eager first call, graph capture on the second, replays
after; plus the pinned copies alone."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import generators as G

for name in ("C4", "C5"):
    cfg = G.CONFIGS[name]
    w, facs = G.cp_config(name)
    pins = []
    for f in facs:  # f: I x R device view; pinned (R, I) host copies
        h = torch.empty(tuple(f.t().shape), dtype=torch.float64, pin_memory=True)
        h.copy_(f.t())
        pins.append(h)
    x = ids.CpTensor(w.cpu().numpy(), [p.numpy().T for p in pins])
    print(name, "pinned views kept:", all(a.base is not None for a in x.factors), flush=True)
    dev = [torch.empty_like(p, device="cuda") for p in pins]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for p, d in zip(pins, dev):
        d.copy_(p, non_blocking=True)
    torch.cuda.synchronize()
    print(f"{name}: pinned copies {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
    for rep in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ids.tensorsketch_id(x, cfg["k"], cfg["L"], seed=rep)
        print(f"{name}: call {rep}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)

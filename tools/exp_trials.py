"""Per-trial time of countsketch_id_sharded_trials on C2 / C3 for pipeline
settings (depth, phase-B grid cap of the background draws), and the single
call.  Usage: python tools/exp_trials.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1901_10559_b200 import generators as G
from paper_1901_10559_b200._inputs import dense_operand
from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials, countsketch_id_sharded

torch.cuda.set_device(0)


def timed(fn, reps=1):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for name in ("C3", "C2"):
    cfg = G.CONFIGS[name]
    a = G.csr_config(name) if name == "C3" else dense_operand(G.dense_config(name))
    rows, k, L = cfg["rows"], cfg["k"], cfg["L"]
    print(name, "single call %.3f ms" % timed(lambda: countsketch_id_sharded(a, 0, rows, k, L, seed=3), 5))
    import time
    for depth, cap, side in ((2, 16, True), (0, 0, True), (2, 0, True), (3, 0, True)):
        t0 = time.perf_counter()
        ms = timed(lambda: countsketch_id_sharded_trials(a, 0, rows, k, L, seeds=range(10),
                                                         depth=depth, grid_cap=cap, id_side=side)) / 10
        host = (time.perf_counter() - t0) / 20 * 1e3
        print(f"  depth {depth} cap {cap} id_side {side}: {ms:.3f} ms per trial (wall {host:.3f})")
    del a
    torch.cuda.empty_cache()

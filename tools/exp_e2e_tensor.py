"""Where the C4/C5 e2e time goes: pinned factor copies alone vs the whole
tensorsketch_id call from host factors."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1901_10559_b200 as ids

for name, N, I, R, k, L in (("C4", 3, 1000, 1000, 10, 4096), ("C5", 4, 10000, 2000, 20, 16384)):
    g = torch.Generator().manual_seed(1)
    facs = [torch.randn(R, I, generator=g, dtype=torch.float64) for _ in range(N)]
    # unit columns, so CpTensor keeps the pinned buffers instead of scaled copies
    pins = [(f / f.norm(dim=1, keepdim=True)).pin_memory() for f in facs]
    w = np.random.default_rng(0).random(R) + 0.5
    x = ids.CpTensor(w, [p.numpy().T for p in pins])
    dev = [torch.empty(R, I, dtype=torch.float64, device="cuda") for _ in range(N)]
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for p, d in zip(pins, dev):
            d.copy_(p, non_blocking=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ids.tensorsketch_id(x, k, L, seed=rep)
        t2 = time.perf_counter()
        nb = sum(p.numel() * 8 for p in pins)
        print(f"{name}: pinned copies {1e3 * (t1 - t0):.2f} ms ({nb / (t1 - t0) / 1e9:.1f} GB/s); "
              f"tensorsketch_id from host {1e3 * (t2 - t1):.2f} ms", flush=True)
    torch.cuda.synchronize()
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        ids.tensorsketch_id(x, k, L, seed=9)
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=14), flush=True)
    prof.export_chrome_trace(f"gpurun_out/trace_{name}.json")

import os, sys, json
sys.path.insert(0, "/root/repo")
import torch
from paper_1901_10559_b200 import generators as G
from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials
op = G.csr_config("C3")
I = op.rows
for _ in range(2):
    countsketch_id_sharded_trials(op, 0, I, 20, 200, seeds=list(range(20)))
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    countsketch_id_sharded_trials(op, 0, I, 20, 200, seeds=list(range(100, 120)))
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/trace_c3_trials.json")

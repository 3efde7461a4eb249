"""Driver for ncu: one warm-up and N full ID calls of a BASELINE config on its
seeded device input (paper_1901_10559_b200.generators), nothing else.

    python tools/prof_config.py --workload C2|C3|C4|C5 [--steps N] [--fortran]

C2 / C3: countsketch_id (device hash, sketch, CPQR, coefficients, j / P to the
host); C4 / C5: tensorsketch_id on device-resident factors (eager path, every
kernel launched from the host)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1901_10559_b200 import generators as G  # noqa: E402
from paper_1901_10559_b200._inputs import dense_operand  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--workload", default="C2", choices=["C2", "C3", "C4", "C5"])
p.add_argument("--steps", type=int, default=1)
p.add_argument("--fortran", action="store_true", help="C2 in column-major layout")
args = p.parse_args()
torch.cuda.set_device(0)
if os.environ.get("IDS_HASH_STAGES"):  # 1: the whole hash chain in one launch (for a kernel capture)
    from paper_1901_10559_b200 import _native

    _native.load().ids_set_hash_stages(int(os.environ["IDS_HASH_STAGES"]), 0)
cfg = G.CONFIGS[args.workload]
if cfg["kind"] in ("dense", "csr"):
    from paper_1901_10559_b200.matrix_id import countsketch_device

    a = (dense_operand(G.dense_config(args.workload, layout="F" if args.fortran else "C"))
         if cfg["kind"] == "dense" else G.csr_config(args.workload))
    torch.cuda.synchronize()
    torch.cuda.profiler.start()  # ncu --profile-from-start off: the ID calls only
    for s in range(args.steps + 1):
        d, _ = countsketch_device(a, cfg["k"], cfg["L"], seed=s, defer_check=True)
        d.to_host("countsketch")
else:
    from paper_1901_10559_b200.distributed import tensorsketch_id_sharded

    w, facs = G.cp_config(args.workload)

    class X:
        factors = facs
        weights = w
        mode_dims = tuple([cfg["dim"]] * cfg["modes"])

    wh = w.cpu().numpy()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for s in range(args.steps + 1):
        tensorsketch_id_sharded(X, 0, cfg["terms"], wh, cfg["k"], cfg["L"], seed=s)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", args.workload)

"""Per-phase timing of the cooperative CPQR kernel on C4/C5-shaped sketches
(debug hook ids_debug_cpqr_timing).  Usage: python tools/exp_cpqr.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1901_10559_b200 as ids
from paper_1901_10559_b200 import _native
from paper_1901_10559_b200.linalg import device_cpqr

lib = _native.load()
lib.ids_debug_cpqr_timing.argtypes = [ctypes.c_void_p]
NAMES = ["pivot col", "sync norm", "gemv", "sync gemv", "F/R columns",
         "recompute", "argmax", "sync step", "hh+z", "z-reduce"]
TALL = ["S1 z loop", "barrier A", "V rows", "gemv", "F/R/downdate", "barrier B", "norm+a loads",
        "hh", "S1 pivot", "S1 y/f loads", "S1 resid+sum", "alpha", "scale", "sykk", "argmax"]


def near_dup(m, n, base, pert, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    b = torch.randn(m, base, generator=g, device="cuda", dtype=torch.float64)
    idx = torch.randint(0, base, (n,), generator=g, device="cuda")
    idx[:base] = torch.arange(base, device="cuda")
    y = b[:, idx] + pert * torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
    return y.t().contiguous()  # (n, m) == col-major m x n


WIDE = ["prologue", "pivot+a", "hh+z", "gemv", "F/R/downdate", "recompute", "publish",
        "barrier"]
CLUSTER = ["pivot select", "pivot col", "householder", "gemv+z", "F/R/downdate",
           "recompute", "argmax", "cluster sync"]
if __name__ != "__main__":
    pass
else:
  for name, m, n, k, base, pert in (("C2", 100, 2000, 20, 20, 1e-2), ("C1", 40, 1000, 10, 10, 1e-2),
                                    ("C4", 4096, 1000, 10, 10, 1e-3),
                                    ("C5", 16384, 2000, 20, 20, 1e-4),
                                    ("C3", 200, 10000, 20, 20, 1e-2)):
      y = near_dup(m, n, base, pert, 1)
      for variant in ("", "old"):
        if variant == "old":
            if m > 1024:
                continue
            os.environ["IDS_CPQR_NO_WIDE"] = "1"
        else:
            os.environ.pop("IDS_CPQR_NO_WIDE", None)
        for _ in range(3):
            device_cpqr(y, m, n, k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            device_cpqr(y, m, n, k)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        buf = torch.zeros(16, dtype=torch.int64, device="cuda")
        lib.ids_debug_cpqr_timing(buf.data_ptr())
        device_cpqr(y, m, n, k)
        torch.cuda.synchronize()
        lib.ids_debug_cpqr_timing(None)
        t = buf.cpu().numpy()
        print(f"{name}{variant}: {m}x{n} k={k}: {ms * 1e3:.1f} us per call; flagged {t[15]}")
        names = TALL if m > 1024 else (WIDE if not variant else (CLUSTER if name in ("C2", "C1") else NAMES))
        for i, nm in enumerate(names):
            print(f"   {nm:14s} {t[i] / 1e3:9.1f} us  ({t[i] / 1e3 / k:6.2f}/step)")

"""Phase clocks of the split-TensorSketch plan builder (library built with
-DIDS_PLAN_TIMING into /tmp/libidsketch_timing.so)."""
import ctypes, os, subprocess, sys
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
csrc = os.path.join(root, "paper_1901_10559_b200", "csrc")
lib_path = "/tmp/libidsketch_timing.so"
subprocess.run(["make", "-s", "-C", csrc, "OBJDIR=/tmp/objt", f"LIB={lib_path}",
                "NVFLAGS=-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC "
                "--expt-relaxed-constexpr -DIDS_PLAN_TIMING"], check=True)
import torch
lib = ctypes.CDLL(lib_path)
N, L = 10000, 16384
torch.manual_seed(0)
bucket = torch.randint(0, L, (N,), dtype=torch.int32, device="cuda")
sign = (torch.randint(0, 2, (N,), dtype=torch.int8, device="cuda") * 2 - 1).to(torch.int8)
lib.ids_ts_split_plan_bytes.restype = ctypes.c_size_t
nb = lib.ids_ts_split_plan_bytes(ctypes.c_int64(N), ctypes.c_int64(L))
plan = torch.empty(nb, dtype=torch.uint8, device="cuda")
args = [ctypes.c_void_p(bucket.data_ptr()), ctypes.c_void_p(sign.data_ptr()), ctypes.c_int64(N),
        ctypes.c_int64(L), ctypes.c_void_p(plan.data_ptr()), ctypes.c_size_t(nb), ctypes.c_void_p(0)]
for _ in range(3):
    lib.ids_ts_split_plan(*args)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 8)()
lib.ids_debug_plan_timing(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    lib.ids_ts_split_plan(*args)
e1.record()
torch.cuda.synchronize()
lib.ids_debug_plan_timing(buf, 0)
print("plan %.1f us" % (e0.elapsed_time(e1) / 10 * 1e3))
for k, nm in enumerate(["load+zero", "walk", "bases", "rank adj", "scan+groups", "codes"]):
    print(f"  {nm:12s} {buf[k] / 10 / 1.9e3:8.2f} us (at 1.9 GHz)")

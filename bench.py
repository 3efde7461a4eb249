"""Benchmark of the CountSketch matrix-ID hot path on B200.

Workload (BASELINE.json configs[1], the largest single-GPU config): dense
fp64 A of 1,000,000 x 2,000 with a rank-20 part and geometric tail
0.9^(i-20) plus N(0, 1e-8) noise; K = 20, CountSketch rows L = 100,
surjective hash.  One step = one countsketch_id of A: device hash draw
(bit-exact numpy PCG64), bucket index, sketch, all-reduce (N > 1), k-step
pivoted QR, triangular solve, and the j / P device->host copy.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Under torchrun (N > 1) the rows are split into N contiguous blocks (strong
scaling: total work fixed) and the L x R sketch is summed with one NCCL
all-reduce.  A (16 GB) is larger than L2 (126 MB), so no flush is needed.
"""

import argparse
import datetime
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: rows, cols, k, L, low rank, tail ratio, noise std
    "C2": dict(rows=1_000_000, cols=2_000, k=20, L=100, lowrank=20, ratio=0.9, noise=1e-4),
    "C1": dict(rows=10_000, cols=1_000, k=10, L=40, lowrank=10, ratio=10 ** -0.1, noise=0.0),
}
METRIC = "sketch HBM GB/s (fraction of B200 peak); matrix ID seconds"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default="C2", choices=sorted(WORKLOADS))
    p.add_argument("--rows", type=int, default=0, help="override rows (debug only)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-rows", type=int, default=200_000)
    p.add_argument("--no-secondary", action="store_true",
                   help="skip the live timings of configs C3-C5")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            m = json.load(fh)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def sigma_of(w):
    i = np.arange(1, w["cols"] + 1, dtype=np.float64)
    return np.where(i <= w["lowrank"], 1.0, w["ratio"] ** (i - w["lowrank"]))


# ----------------------------------------------------------------- inputs --
CHUNK = 125_000  # global rows per generator chunk (so A is identical for any N | 8)


def make_rows_device(w, r0, r1, torch, dev):
    """Rows [r0, r1) of A = U diag(sigma) V^T + noise, generated on the GPU.

    U's rows are N(0, 1/rows) (columns orthonormal up to O(1/sqrt(rows))),
    V is the Q factor of a seeded 2000 x 2000 Gaussian, both seeded per fixed
    global chunk so every rank builds the same global matrix."""
    cols = w["cols"]
    g = torch.Generator(device=dev)
    g.manual_seed(1234)
    v = torch.linalg.qr(torch.randn(cols, cols, generator=g, device=dev, dtype=torch.float64))[0]
    vs = (v * torch.from_numpy(sigma_of(w)).to(dev)).t().contiguous()  # diag(s) V^T
    out = torch.empty((r1 - r0, cols), dtype=torch.float64, device=dev)
    c = (r0 // CHUNK) * CHUNK
    while c < r1:
        c1 = min(c + CHUNK, w["rows"])
        g.manual_seed(10_000 + c // CHUNK)
        u = torch.randn(c1 - c, cols, generator=g, device=dev, dtype=torch.float64)
        u /= float(np.sqrt(w["rows"]))
        blk = u @ vs
        if w["noise"] > 0:
            blk += w["noise"] * torch.randn(c1 - c, cols, generator=g, device=dev,
                                            dtype=torch.float64)
        a, b = max(c, r0), min(c1, r1)
        out[a - r0:b - r0] = blk[a - c:b - c]
        del u, blk
        c = c1
    return out


# ----------------------------------------------------------------- clocks --
class Clocks:
    def __init__(self, enabled):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        self.t0 = time.time()
        if not enabled:
            return
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self, gpu_index, window=None):
        """Median SM clock, max clock and throttle reasons of the samples taken
        inside `window` (wall-clock seconds, time.time()) when given."""
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 10:
                continue
            if window is not None:
                try:
                    ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    continue
                if not window[0] <= ts <= window[1]:
                    continue
            f = f[1:]
            if not f[0].isdigit() or int(f[0]) != gpu_index:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)),
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- CPU -----
def cpu_sample_matrix(w, rows):
    """A row sample of the workload built the same way (host numpy)."""
    rng = np.random.default_rng(7)
    cols = w["cols"]
    v = np.linalg.qr(rng.standard_normal((cols, cols)))[0]
    u = rng.standard_normal((rows, cols)) / np.sqrt(w["rows"])
    a = (u * sigma_of(w)) @ v.T
    if w["noise"] > 0:
        a += w["noise"] * rng.standard_normal(a.shape)
    # F order, as BASELINE.md section 2 prescribes for the reference (no extra copy
    # in as_dense, linalg.py:29)
    return np.asfortranarray(a)


def cpu_sample_gbs(w, rows, seed=0, a=None):
    """The oracle port (reference algorithm on numpy/scipy/LAPACK) on a
    bounded row sample of the workload; returns (GB/s, seconds, rows)."""
    import oracle

    if a is None:
        a = cpu_sample_matrix(w, rows)
    t0 = time.perf_counter()
    oracle.countsketch_id(a, w["k"], w["L"], seed=seed)
    dt = time.perf_counter() - t0
    return a.nbytes / dt / 1e9, dt, a.shape[0]


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, w, rank, world):
    if rank != 0:
        return
    rows = min(args.cpu_rows, w["rows"])
    a = cpu_sample_matrix(w, rows)
    vals = []
    for step in range(args.warmup + args.steps):
        gbs, dt, _ = cpu_sample_gbs(w, rows, seed=step, a=a)
        if step >= args.warmup:
            vals.append((gbs, dt))
    gb = float(np.median([v[0] for v in vals]))
    sec = float(np.median([v[1] for v in vals]))
    sample = (f"{rows} x {w['cols']} row sample of {args.workload} "
              f"({rows * w['cols'] * 8 / 1e9:.2f} GB), full countsketch_id")
    line = {
        "impl": "reference", "metric": METRIC, "value": gb, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(args, w, world),
        "cpu_baseline": {"value": gb, "unit": "GB/s", "cores": cores(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": gb, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_of(args, w, world):
    rows = args.rows or w["rows"]
    return {"workload": f"{args.workload}: dense fp64 {rows}x{w['cols']} countsketch_id "
                        f"K={w['k']} L={w['L']} surjective",
            "rows": rows, "cols": w["cols"], "rank": w["k"], "sketch_dim": w["L"],
            "parallelism": f"rows{world}", "l2": "A (>126 MB) larger than L2, no flush"}


def secondary_configs(torch, dev, steps=6):
    """Live device timings (CUDA events, after warm-up) of one full ID at the
    other BASELINE.json configs, on seeded synthetic inputs of their shapes
    built on the device: C3 CSR 1e7 x 1e4 with 1e8 nonzeros,
    C4 / C5 CP tensors with near-duplicate terms.  Reported beside the
    headline, not part of it."""
    import paper_1901_10559_b200 as ids
    from paper_1901_10559_b200._inputs import SparseOperand
    from paper_1901_10559_b200.matrix_id import countsketch_device, device_matrix_id

    def timed(fn):
        for s in range(2):
            fn(10_000 + s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in range(steps):
            fn(20_000 + s)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    out = {}
    g = torch.Generator(device=dev).manual_seed(3)
    I, R, per, K, L = 10_000_000, 10_000, 10, 20, 200
    indptr = torch.arange(0, I + 1, dtype=torch.int64, device=dev) * per
    idx = torch.randint(0, R, (I, per), generator=g, device=dev).sort(dim=1).values
    idx = idx.to(torch.int32).reshape(-1)
    data = torch.randn(I * per, generator=g, device=dev, dtype=torch.float64)
    csr = SparseOperand("csr", indptr, idx, data, I, R, I * per)
    ms = timed(lambda s: countsketch_device(csr, K, L, seed=s)[0].to_host("countsketch"))
    nbytes = int(I * per * 12 + (I + 1) * 8)
    # the sketch kernel alone (hash drawn once, outside the clock)
    op = ids.CountSketchOp(I, L, seed=1, surjective=True)
    y = torch.empty((R, L), dtype=torch.float64, device=dev)
    sk_ms = timed(lambda s: op.sketch_into(csr, y, flags=0))
    out["C3"] = {"id_ms": ms, "shape": "CSR 1e7 x 1e4, nnz 1e8 (10 per row), K=20, L=200",
                 "algorithmic_bytes": nbytes,
                 "sketch": {"kernel": "cs_csr_stream_kernel", "ms": sk_ms,
                            "achieved_gbs": nbytes / sk_ms / 1e6,
                            "bound": "L2 fp64 reductions (one per nonzero)"}}
    del op, y
    del indptr, idx, data, csr
    for name, N, In, R, base, pert, K, L in (("C4", 3, 1000, 1000, 10, 1e-3, 10, 4096),
                                             ("C5", 4, 10_000, 2000, 20, 1e-4, 20, 16384)):
        g = torch.Generator(device=dev).manual_seed(4 if name == "C4" else 5)
        bases = torch.randint(0, base, (R,), generator=g, device=dev)
        bases[:base] = torch.arange(base, device=dev)
        facs = []
        for _ in range(N):
            f = torch.randn(In, R, generator=g, device=dev, dtype=torch.float64)
            f[:, :base] /= torch.linalg.vector_norm(f[:, :base], dim=0)
            f = f[:, bases] + pert * torch.randn(In, R, generator=g, device=dev,
                                                 dtype=torch.float64)
            f /= torch.linalg.vector_norm(f, dim=0)
            facs.append(f.t().contiguous().t())  # column-major I_n x R
        w = torch.rand(R, generator=g, device=dev, dtype=torch.float64) * 0.5 + 0.5

        def step(s, facs=facs, w=w, N=N, In=In, R=R, K=K, L=L):
            y = ids.TensorSketchOp([In] * N, L, seed=s).apply_device(facs, w)
            return device_matrix_id(y, L, R, K).to_host("tensorsketch")

        out[name] = {"id_ms": timed(step),
                     "shape": f"CP N={N}, I_n={In}, R={R}, K={K}, L={L}, near-duplicate terms",
                     "algorithmic_bytes": int(N * In * R * 8)}
        del facs
    return out


# ----------------------------------------------------------------- GPU -----
def prime_nvml():
    """One nvidia-smi call at start-up: the driver/NVML initialization it can
    trigger lands long before anything is timed."""
    try:
        subprocess.run(["nvidia-smi", "-q", "-d", "CLOCK"], capture_output=True, timeout=120)
    except Exception:
        pass


def main():
    args = parse()
    w = dict(WORKLOADS[args.workload])
    if args.rows:
        w["rows"] = args.rows
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, w, rank, world)

    if local == 0:
        prime_nvml()
    import torch
    import torch.distributed as dist

    # IDS_BENCH_ONE_DEVICE=1 (test hook): every rank on cuda:0 over gloo, which
    # stages collectives through the host -- exercises the multi-rank code
    # path on a one-GPU box; its timings mean nothing
    one_dev = os.environ.get("IDS_BENCH_ONE_DEVICE") == "1"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    import paper_1901_10559_b200 as ids
    from paper_1901_10559_b200 import _native
    from paper_1901_10559_b200._inputs import dense_operand
    from paper_1901_10559_b200.distributed import countsketch_id_sharded, row_block
    from paper_1901_10559_b200.matrix_id import device_matrix_id

    lib = _native.load()
    r0, r1 = row_block(w["rows"], world, rank)
    a_dev = make_rows_device(w, r0, r1, torch, dev)
    torch.cuda.synchronize()
    operand = dense_operand(a_dev)
    bytes_local = a_dev.numel() * 8
    bytes_total = w["rows"] * w["cols"] * 8

    def barrier():
        if world > 1:
            dist.barrier()

    from paper_1901_10559_b200.distributed import DeviceBackend

    backend = DeviceBackend()

    def step(seed):
        return countsketch_id_sharded(operand, r0, w["rows"], w["k"], w["L"], seed=seed,
                                      backend=backend)

    # ---- single-call latency (no cross-trial overlap): the ID seconds ----
    for s in range(2):
        step(s)
    torch.cuda.synchronize()
    barrier()
    t_single = []
    for s in range(3):
        e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_a.record()
        step(100 + s)
        e_b.record()
        torch.cuda.synchronize()
        t_single.append(e_a.elapsed_time(e_b))
    single_ms = float(np.median(t_single))

    from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials

    # ---- device-resident steps (value): K trials queued back to back ----
    # warm-up: at least as many trials as one timed batch, so the allocator
    # already holds every buffer a batch needs (no cudaMalloc while timed)
    countsketch_id_sharded_trials(operand, r0, w["rows"], w["k"], w["L"],
                                  seeds=list(range(max(args.warmup, args.steps))))
    torch.cuda.synchronize()
    # the clock sampler runs under load: started here (its start-up lands in an
    # idle second), then untimed trials for about a second before and after
    # the timed batch; only samples from that busy window are reported
    clocks = Clocks(rank == 0)
    time.sleep(1.0)
    busy0 = time.time()
    while time.time() - busy0 < 1.0:
        countsketch_id_sharded_trials(operand, r0, w["rows"], w["k"], w["L"],
                                      seeds=list(range(args.steps)))
    torch.cuda.synchronize()
    barrier()
    n0 = lib.ids_launch_count()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier()
    start.record()
    ds = countsketch_id_sharded_trials(operand, r0, w["rows"], w["k"], w["L"],
                                       seeds=[1000 + s for s in range(args.steps)])
    d = ds[-1]
    stop.record()
    torch.cuda.synchronize()
    barrier()
    launches = (lib.ids_launch_count() - n0) // max(args.steps, 1)
    ms = start.elapsed_time(stop) / args.steps
    busy1 = time.time()
    while time.time() - busy1 < 1.0:
        countsketch_id_sharded_trials(operand, r0, w["rows"], w["k"], w["L"],
                                      seeds=list(range(args.steps)))
    torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clk = clocks.stop(local, window=(busy0, time.time()))

    # ---- dominant kernel alone: the sketch (roofline) ----
    op = ids.CountSketchOp(w["rows"], w["L"], seed=5, surjective=True)
    y = torch.empty((w["cols"], w["L"]), dtype=torch.float64, device=dev)
    op.bucket_index()
    for _ in range(2):
        op.sketch_into(operand, y, row0=r0, flags=1)
    torch.cuda.synchronize()
    reps = max(3, args.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        op.sketch_into(operand, y, row0=r0, flags=1)
    e1.record()
    torch.cuda.synchronize()
    sk_ms = e0.elapsed_time(e1) / reps
    # CPQR + coefficients alone (ID seconds without the sketch)
    e0.record()
    for _ in range(reps):
        device_matrix_id(y, w["L"], w["cols"], w["k"])
    e1.record()
    torch.cuda.synchronize()
    id_ms = e0.elapsed_time(e1) / reps
    # hash draw alone
    e0.record()
    for s in range(reps):
        ids.CountSketchOp(w["rows"], w["L"], seed=s, surjective=True).bucket_index()
    e1.record()
    torch.cuda.synchronize()
    hash_ms = e0.elapsed_time(e1) / reps

    peak, peak_kind = peaks()
    achieved = bytes_local / (sk_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.workload)
        except Exception:
            traffic = None
    if traffic is not None and world > 1:
        # the capture is of the whole-matrix launch (one GPU): scale to this
        # rank's row block by the measured traffic / algorithmic-bytes ratio
        traffic = traffic * bytes_local / bytes_total

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        try:
            host = torch.empty((r1 - r0, w["cols"]), dtype=torch.float64, pin_memory=True)
            host.copy_(a_dev, non_blocking=False)
            del_dev = True
        except RuntimeError:
            host, del_dev = None, False
        if host is not None:
            def api(seed):
                if world == 1:  # the call a user makes
                    return ids.countsketch_id(host, w["k"], w["L"], seed=seed)
                return countsketch_id_sharded(host, r0, w["rows"], w["k"], w["L"], seed=seed)

            d = api(1)
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            e0.record()
            nsteps = max(1, min(args.steps, 3))
            for s in range(nsteps):
                d = api(2000 + s)
            e1.record()
            torch.cuda.synchronize()
            e2e_ms = e0.elapsed_time(e1) / nsteps
            if world > 1:
                t = torch.tensor([e2e_ms], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                e2e_ms = float(t.item())
            e2e = {"value": bytes_total / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
                   "h2d_bytes_per_step": bytes_total,
                   "d2h_bytes_per_step": int(d.coeffs.nbytes + d.cols.nbytes) * world,
                   "ms_per_step": e2e_ms, "wall_s": time.perf_counter() - t0}
            del host
            _ = del_dev

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        gbs, dt, rows = cpu_sample_gbs(w, min(args.cpu_rows, w["rows"]))
        cpu = {"value": gbs, "unit": "GB/s", "cores": cores(), "kind": "port",
               "sample": f"{rows} x {w['cols']} row sample of {args.workload}, full "
                         f"countsketch_id in {dt:.2f} s (scipy S@A single-threaded, "
                         f"LAPACK dgeqp3 multithreaded)"}

    secondary = None
    if rank == 0 and world == 1 and not args.no_secondary:
        del a_dev, operand
        torch.cuda.empty_cache()
        secondary = secondary_configs(torch, dev)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": bytes_total / (ms * 1e-3) / 1e9,
            "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_of(args, w, world),
            "id_seconds": single_ms * 1e-3,
            "trials": ("K trials (seeds) of the same A queued back to back, one host sync at "
                       "the end; each trial's hash is drawn on the device on a side stream "
                       "beside the earlier trials' sketches (sketch.pipelined_operators)"
                       if world == 1 else
                       "K trials (seeds) of the same row-sharded A queued back to back, one "
                       "host sync at the end; trial t's hash is drawn by rank t mod N and "
                       "broadcast (distributed.trial_sharded_operators), each rank sketches "
                       "its rows, one all-reduce of the sketch per trial"),
            "phases_ms": {"hash_and_index": hash_ms, "sketch": sk_ms, "cpqr_and_coeffs": id_ms},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "cs_rowmajor_kernel", "peak_kind": peak_kind,
                         "bytes_per_launch": bytes_local},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "secondary_configs": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

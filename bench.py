"""Benchmark of the CountSketch / TensorSketch ID hot path on B200.

    python bench.py [--gpus N --steps K --warmup W] [--workload C2|C3|C4|C5]
                    [--impl b200|reference]

Workloads are BASELINE.json's configs, built on the device by
``paper_1901_10559_b200.generators`` (seeded synthetic inputs of the stated
shapes and value distributions -- the paper's SuiteSparse / FROSTT data is
not available offline):

* C2 (default, the headline): dense fp64 1,000,000 x 2,000, K = 20, L = 100,
  surjective CountSketch; rows sharded over the ranks, one all-reduce of the
  L x R sketch per trial.
* C3: CSR 1e7 x 1e4, ~1e8 nonzeros, planted latent rank-20 structure,
  K = 20, L = 200; rows sharded.
* C4 / C5: CP tensors (N = 3, I = 1e3, R = 1e3, L = 4096 / N = 4, I = 1e4,
  R = 2e3, L = 16384) with near-duplicate terms; terms sharded, the ID by
  the column-distributed truncated CPQR.

One step = one full ID trial (hash draw, sketch, collective, pivoted QR,
coefficients, j / P to the host) on device-resident input; `value` = the
workload's algorithmic bytes (A, or the factor matrices, read once) per
step time, whole job.  Total work is fixed as N grows ("strong").  The
headline line also carries the other configs (`secondary_configs`), each
with its own roofline, CPU baseline, parity and end-to-end numbers at N = 1.

With --gpus N > 1 outside torchrun the script re-launches itself under
``torch.distributed.run`` (one process per GPU, NCCL).
"""

import argparse
import datetime
import json
import os
import socket
import subprocess
import sys
import time

_REF_ARM = "--impl=reference" in sys.argv or any(
    a == "--impl" and b == "reference" for a, b in zip(sys.argv, sys.argv[1:]))
if _REF_ARM and "TORCHELASTIC_RUN_ID" in os.environ and os.environ.get("OMP_NUM_THREADS") == "1":
    # torch.distributed.run pins OMP_NUM_THREADS=1 in every rank; the
    # reference arm's rank 0 is a CPU job that should use the host's cores
    # (LAPACK / OpenBLAS read it when numpy loads, just below)
    del os.environ["OMP_NUM_THREADS"]

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

METRIC = "sketch HBM GB/s (fraction of B200 peak); matrix/tensor ID seconds at 1/2/4/8 GPU"
CPU_SAMPLE_ROWS = 200_000  # C2's CPU legs run on this many leading rows of A
FP64_PEAK_DATASHEET = 37.0  # TFLOP/s, B200 fp64 (non-tensor) datasheet figure


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default="C2", choices=["C2", "C3", "C4", "C5"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true", help="skip the CPU baselines / parity")
    p.add_argument("--no-secondary", action="store_true", help="headline workload only")
    p.add_argument("--cpu-rows", type=int, default=CPU_SAMPLE_ROWS)
    return p.parse_args()


def maybe_spawn(args):
    """--gpus N > 1 outside torchrun: re-launch under torch.distributed.run."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def relerr(got, want):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    den = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / (den if den > 0 else 1.0))


# ------------------------------------------------------- CPU reference -----
class RefCPU:
    """The reference's own CPU implementation of the path: the unmodified
    ``idsketch`` package installed in baseline/_ref when present (kind
    "reference"), else the oracle port (numpy/scipy/LAPACK restatement,
    kind "port").  Each call runs the steps of countsketch_id /
    tensorsketch_id (matrix_id.py:162-182, cp_tensor.py:266-276) and also
    returns the sketch for the parity check."""

    def __init__(self):
        self.kind = "port"
        try:
            if os.path.isdir(os.path.join(REF_DIR, "idsketch")):
                sys.path.insert(0, REF_DIR)
                import idsketch  # noqa: F401

                self.ref = idsketch
                self.kind = "reference"
        except Exception:
            self.kind = "port"
        if self.kind == "port":
            import oracle

            self.ref = oracle

    def matrix(self, a, k, L, seed):
        import scipy.sparse as sp

        t0 = time.perf_counter()
        if self.kind == "reference":
            from idsketch.linalg import as_csc, as_dense
            from idsketch.matrix_id import matrix_id, matrix_sketch

            a2 = as_csc(a) if sp.issparse(a) else as_dense(a)
            y = matrix_sketch(a2, "countsketch", L, seed=seed, surjective=True)
            d = matrix_id(y, k)
        else:
            d = self.ref.countsketch_id(a, k, L, seed=seed)
            y = d.sketch
        dt = time.perf_counter() - t0
        return {"s": dt, "cols": np.asarray(d.cols), "coeffs": np.asarray(d.coeffs), "y": y}

    def tensor(self, weights, factors, k, L, seed):
        if self.kind == "reference":
            x = self.ref.CpTensor(weights, factors)
            t0 = time.perf_counter()
            op = self.ref.TensorSketchOp(x.mode_dims, L, seed=seed)
            y = op.apply(x.factors, x.weights)
            from idsketch.cp_tensor import tensor_id_from_sketch

            res = tensor_id_from_sketch(x, y, k, "tensorsketch")
            dt = time.perf_counter() - t0
            return {"s": dt, "cols": res.cols, "coeffs": res.coeffs, "y": y,
                    "new_weights": res.new_weights}
        t0 = time.perf_counter()
        d, nw = self.ref.tensorsketch_id(weights, factors, k, L, seed=seed)
        dt = time.perf_counter() - t0
        return {"s": dt, "cols": d.cols, "coeffs": d.coeffs, "y": d.sketch, "new_weights": nw}


def host_sample_c2(rows, cols=2000, seed=7):
    """Host-only stand-in for a row block of C2 (the reference arm must not
    touch the product): rows of U are N(0, 1/1e6) (a 1e6-row orthonormal U's
    rows up to O(1e-3)), the same sigma and noise as generators.dense_config."""
    rng = np.random.default_rng(seed)
    i = np.arange(1, cols + 1, dtype=np.float64)
    sig = np.where(i <= 20, 1.0, 0.9 ** (i - 20))
    v = np.linalg.qr(rng.standard_normal((cols, cols)))[0]
    a = (rng.standard_normal((rows, cols)) / 1e3 * sig) @ v.T
    a += 1e-4 * rng.standard_normal(a.shape)
    return np.asfortranarray(a)


def config_of(name, world, cpu_rows=CPU_SAMPLE_ROWS):
    from_cfg = {
        "C2": dict(shape="dense fp64 1000000x2000", k=20, L=100, parallelism=f"rows{world}",
                   cpu_sample=f"{cpu_rows} leading rows (F order)"),
        "C3": dict(shape="CSR fp64 10000000x10000, ~1e8 nnz, planted latent rank 20", k=20,
                   L=200, parallelism=f"rows{world}", cpu_sample="full matrix"),
        "C4": dict(shape="CP N=3 I_n=1000 R=1000 near-duplicate terms", k=10, L=4096,
                   parallelism=f"terms{world}", cpu_sample="full tensor"),
        "C5": dict(shape="CP N=4 I_n=10000 R=2000 near-duplicate terms", k=20, L=16384,
                   parallelism=f"terms{world}", cpu_sample="full tensor"),
    }[name]
    kind = "countsketch_id surjective" if name in ("C2", "C3") else "tensorsketch_id"
    out = {"workload": f"{name}: {from_cfg['shape']} {kind} K={from_cfg['k']} L={from_cfg['L']}"}
    out.update(from_cfg)
    out["l2"] = ("inputs larger than the 126 MB L2, no flush" if name != "C4" else
                 "C4 factors (24 MB) fit in L2: steps run back to back, no flush "
                 "(the reference config is that small)")
    return out


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation on this box's host
    cores, rank 0 only, each step a bounded sample of the workload."""
    if rank != 0:
        return
    ref = RefCPU()
    name = args.workload
    if name == "C2":
        a = host_sample_c2(min(args.cpu_rows, 1_000_000))
        nbytes = a.nbytes
        run = lambda s: ref.matrix(a, 20, 100, s)  # noqa: E731
        sample = f"{a.shape[0]} x {a.shape[1]} row sample of C2 ({nbytes / 1e9:.2f} GB), F order"
    else:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"reference arm is timed on the headline workload C2 only (got {name})"}))
        return
    secs = []
    for step in range(args.warmup + args.steps):
        r = run(step)
        if step >= args.warmup:
            secs.append(r["s"])
    sec = float(np.median(secs))
    gbs = nbytes / sec / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(name, world, args.cpu_rows),
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores(), "kind": ref.kind,
                         "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- clocks --
class Clocks:
    """nvidia-smi sampler (100 ms) around the timed region."""

    def __init__(self, enabled):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
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


def prime_nvml():
    try:
        subprocess.run(["nvidia-smi", "-q", "-d", "CLOCK"], capture_output=True, timeout=120)
    except Exception:
        pass


# -------------------------------------------------------------- workloads --
class Ctx:
    """Per-process device / collective context."""

    def __init__(self, torch, dist, dev, rank, world):
        self.torch, self.dist, self.dev, self.rank, self.world = torch, dist, dev, rank, world

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max_over_ranks(self, v):
        if self.world == 1:
            return float(v)
        t = self.torch.tensor([float(v)], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, v):
        if self.world == 1:
            return float(v)
        t = self.torch.tensor([float(v)], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t)
        return float(t.item())

    def events(self, fn, reps):
        """Average device time (ms) of fn() over reps calls, CUDA events on the
        current stream, synchronized on both sides."""
        torch = self.torch
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for i in range(reps):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps


class MatrixWorkload:
    """C2 (dense) / C3 (CSR): rows [r0, r1) of A on this rank."""

    def __init__(self, ctx, name):
        from paper_1901_10559_b200 import generators as G
        from paper_1901_10559_b200._inputs import dense_operand
        from paper_1901_10559_b200.distributed import row_block

        self.ctx, self.name = ctx, name
        cfg = G.CONFIGS[name]
        self.rows, self.cols, self.k, self.L = cfg["rows"], cfg["cols"], cfg["k"], cfg["L"]
        self.r0, self.r1 = row_block(self.rows, ctx.world, ctx.rank)
        if cfg["kind"] == "dense":
            self.operand = dense_operand(G.dense_config(name, row_range=(self.r0, self.r1)))
            self.bytes_local = (self.r1 - self.r0) * self.cols * 8
            self.kernel_name = "cs_rowmajor_kernel"
        else:
            self.operand = G.csr_config(name, row_range=(self.r0, self.r1))
            ptr_b = self.operand.indptr.element_size()
            self.bytes_local = self.operand.nnz * 12 + (self.r1 - self.r0 + 1) * ptr_b
            self.kernel_name = "cs_csr_stream_kernel"
        ctx.torch.cuda.synchronize()
        self.bytes_total = int(ctx.sum_over_ranks(self.bytes_local))

    def bytes_note(self):
        if self.name == "C2":
            return "8 B per element of A (1e6 x 2000 fp64)"
        return "12 B per nonzero (fp64 value + int32 column) + 4 B per row pointer"

    def trials(self, seeds):
        from paper_1901_10559_b200.distributed import countsketch_id_sharded_trials

        return countsketch_id_sharded_trials(self.operand, self.r0, self.rows, self.k, self.L,
                                             seeds=list(seeds))

    def single(self, seed):
        from paper_1901_10559_b200.distributed import countsketch_id_sharded

        return countsketch_id_sharded(self.operand, self.r0, self.rows, self.k, self.L,
                                      seed=seed)

    def kernel(self, reps):
        """The sketch kernel alone: (ms per launch, bytes per launch, extra)."""
        import paper_1901_10559_b200 as ids

        torch = self.ctx.torch
        op = ids.CountSketchOp(self.rows, self.L, seed=5, surjective=True)
        op.bucket_index()
        y = torch.empty((self.cols, self.L), dtype=torch.float64, device=self.ctx.dev)
        flags = 1 if self.name == "C2" else 0
        for _ in range(2):
            op.sketch_into(self.operand, y, row0=self.r0, flags=flags)
        ms = self.ctx.events(lambda i: op.sketch_into(self.operand, y, row0=self.r0,
                                                      flags=flags), reps)
        from paper_1901_10559_b200.matrix_id import device_matrix_id

        device_matrix_id(y, self.L, self.cols, self.k)
        id_ms = self.ctx.events(lambda i: device_matrix_id(y, self.L, self.cols, self.k), reps)
        # one untimed draw first: its workspace comes from the caching allocator afterwards
        ids.CountSketchOp(self.rows, self.L, seed=99, surjective=True).bucket_index()
        hash_ms = self.ctx.events(lambda i: ids.CountSketchOp(
            self.rows, self.L, seed=100 + i, surjective=True).bucket_index(), reps)
        return ms, self.bytes_local, {"cpqr_and_coeffs": id_ms, "hash_and_index": hash_ms}

    def host_copy(self):
        """This rank's block in pinned host memory: a pinned tensor (dense) or a
        scipy CSR over pinned arrays (the contract's e2e input)."""
        torch = self.ctx.torch
        if self.operand.kind == "dense":
            h = torch.empty((self.r1 - self.r0, self.cols), dtype=torch.float64, pin_memory=True)
            h.copy_(self.operand.t)
            return h, int(h.numel() * 8)
        import scipy.sparse as sp

        parts = [pinned_copy(torch, t) for t in (self.operand.data, self.operand.indices,
                                                 self.operand.indptr)]
        m = sp.csr_array(tuple(p.numpy() for p in parts), shape=self.operand.shape)
        m._pinned = parts  # keep the pinned buffers alive with the matrix
        return m, int(sum(p.numel() * p.element_size() for p in parts))

    def e2e_call(self, host, seed):
        import paper_1901_10559_b200 as ids
        from paper_1901_10559_b200.distributed import countsketch_id_sharded

        if self.ctx.world == 1:  # the call a user makes
            return ids.countsketch_id(host, self.k, self.L, seed=seed)
        return countsketch_id_sharded(host, self.r0, self.rows, self.k, self.L, seed=seed)

    def cpu_and_parity(self, ref, cpu_rows, seed=11):
        """The reference on the host (C2: leading rows, C3: the full matrix)
        and the product on the same input and seed."""
        import paper_1901_10559_b200 as ids

        if self.name == "C2":
            rows = min(cpu_rows, self.rows)
            a = np.asfortranarray(self.operand.t[:rows].cpu().numpy())
            sample = f"{rows} x {self.cols} leading rows of C2 ({a.nbytes / 1e9:.2f} GB), F order"
            nbytes = a.nbytes
        else:
            from paper_1901_10559_b200.generators import operand_to_scipy

            a = operand_to_scipy(self.operand)
            rows = self.rows
            sample = f"full C3 matrix ({a.nnz} nonzeros)"
            nbytes = self.bytes_local
        r = ref.matrix(a, self.k, self.L, seed)
        d = ids.countsketch_id(a, self.k, self.L, seed=seed)
        y = ids.CountSketchOp(rows, self.L, seed=seed, surjective=True).apply(a)
        cpu = {"value": nbytes / r["s"] / 1e9, "unit": "GB/s", "cores": cores(),
               "kind": ref.kind, "seconds": r["s"],
               "sample": sample + ", full countsketch_id (as_dense/as_csc, S@A, dgeqp3, dtrtrs)"}
        parity = {"input": sample, "seed": seed,
                  "cols_equal": bool(np.array_equal(d.cols, r["cols"])),
                  "P_relerr": relerr(d.coeffs, r["coeffs"]),
                  "Y_relerr": relerr(y, r["y"]),
                  "Y_bit_exact": bool(np.array_equal(y, r["y"])),
                  "against": ref.kind}
        return cpu, parity


class TensorWorkload:
    """C4 / C5: terms [c0, c1) of the CP tensor on this rank."""

    def __init__(self, ctx, name):
        from paper_1901_10559_b200 import generators as G
        from paper_1901_10559_b200.distributed import row_block

        self.ctx, self.name = ctx, name
        cfg = G.CONFIGS[name]
        self.N, self.I, self.R, self.k, self.L = (cfg["modes"], cfg["dim"], cfg["terms"],
                                                  cfg["k"], cfg["L"])
        self.c0, self.c1 = row_block(self.R, ctx.world, ctx.rank)
        w, facs = G.cp_config(name)
        self.w_all = w.cpu().numpy()
        self.w_local = w[self.c0:self.c1].contiguous()
        self.f_local = [f[:, self.c0:self.c1] for f in facs]  # column-major views
        self.full = (w, facs) if ctx.world == 1 else None
        self.bytes_local = self.N * self.I * (self.c1 - self.c0) * 8
        self.bytes_total = self.N * self.I * self.R * 8
        self.flops_local = (self.N + 1) * (self.c1 - self.c0) * 2.5 * self.L * np.log2(self.L)
        from paper_1901_10559_b200.tensorsketch import uses_split_kernel

        self.kernel_name = ("ts_split_kernel" if uses_split_kernel(self.N, self.L)
                            else "tensorsketch_kernel")
        self.graph = None

        class _X:
            factors = self.f_local
            weights = self.w_local
            mode_dims = tuple([self.I] * self.N)

        self.x_local = _X

    def bytes_note(self):
        return (f"8 B per factor entry ({self.N} x {self.I} x {self.R} fp64); fp64 FFT work "
                f"(N+1) x R x 2.5 L log2 L flops")

    def _graph(self):
        if self.graph is None:
            import paper_1901_10559_b200 as ids

            self.graph = ids.TensorIdGraph(self.f_local, self.w_local, self.k, self.L,
                                           host_weights=self.w_all)
        return self.graph

    def trials(self, seeds):
        if self.ctx.world == 1:  # replays of the captured CUDA graph, one sync
            return self._graph().trials(seeds)
        from paper_1901_10559_b200.distributed import tensorsketch_id_sharded_trials

        return tensorsketch_id_sharded_trials(self.x_local, self.c0, self.R, self.w_all,
                                              self.k, self.L, seeds=list(seeds))

    def single(self, seed):
        if self.ctx.world == 1:  # one call = one replay of the captured CUDA graph
            return self._graph()(seed)
        from paper_1901_10559_b200.distributed import tensorsketch_id_sharded

        return tensorsketch_id_sharded(self.x_local, self.c0, self.R, self.w_all, self.k,
                                       self.L, seed=seed)

    def kernel(self, reps):
        import paper_1901_10559_b200 as ids
        from paper_1901_10559_b200.matrix_id import device_matrix_id

        op = ids.TensorSketchOp([self.I] * self.N, self.L, seed=5)
        y = op.apply_device(self.f_local, self.w_local)
        ms = self.ctx.events(lambda i: op.apply_device(self.f_local, self.w_local), reps)
        n_loc = self.c1 - self.c0
        device_matrix_id(y, self.L, n_loc, self.k)
        id_ms = self.ctx.events(lambda i: device_matrix_id(y, self.L, n_loc, self.k), reps)
        return ms, self.bytes_local, {"cpqr_and_coeffs_local_block": id_ms,
                                      "flops_per_launch": self.flops_local,
                                      "y_write_bytes": n_loc * self.L * 8}

    def host_copy(self):
        """The CP tensor over factors in pinned host memory (F order)."""
        import paper_1901_10559_b200 as ids

        torch = self.ctx.torch
        w = self.w_local.cpu().numpy()
        pins = [pinned_copy(torch, f.t()) for f in self.f_local]  # (R, I_n) contiguous
        x = ids.CpTensor(w, [p.numpy().T for p in pins])  # I_n x R, F order, no copy
        x._pinned = pins
        return x, int(sum(p.numel() * 8 for p in pins) + w.nbytes)

    def e2e_call(self, host, seed):
        import paper_1901_10559_b200 as ids
        from paper_1901_10559_b200.distributed import tensorsketch_id_sharded

        if self.ctx.world == 1:
            return ids.tensorsketch_id(host, self.k, self.L, seed=seed)
        return tensorsketch_id_sharded(host, self.c0, self.R, self.w_all, self.k, self.L,
                                       seed=seed)

    def cpu_and_parity(self, ref, cpu_rows, seed=11):
        import paper_1901_10559_b200 as ids

        w, facs = self.full
        wh = w.cpu().numpy()
        fh = [f.cpu().numpy() for f in facs]
        r = ref.tensor(wh, fh, self.k, self.L, seed)
        x = ids.CpTensor(wh, fh)
        res = ids.tensorsketch_id(x, self.k, self.L, seed=seed)
        y = ids.TensorSketchOp(x.mode_dims, self.L, seed=seed).apply(x.factors, x.weights)
        sample = f"full {self.name} tensor ({self.bytes_total / 1e6:.0f} MB of factors)"
        cpu = {"value": self.bytes_total / r["s"] / 1e9, "unit": "GB/s", "cores": cores(),
               "kind": ref.kind, "seconds": r["s"],
               "sample": sample + ", full tensorsketch_id (CountSketch, pocketfft, dgeqp3)"}
        parity = {"input": sample, "seed": seed,
                  "cols_equal": bool(np.array_equal(res.cols, r["cols"])),
                  "P_relerr": relerr(res.coeffs, r["coeffs"]),
                  "Y_relerr": relerr(y, r["y"]),
                  "new_weights_relerr": relerr(res.new_weights, r["new_weights"]),
                  "against": ref.kind}
        return cpu, parity


def pinned_copy(torch, t):
    """A pinned host copy of device tensor t (same shape, contiguous)."""
    h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h


def make_workload(ctx, name):
    return MatrixWorkload(ctx, name) if name in ("C2", "C3") else TensorWorkload(ctx, name)


def fp64_peak(ctx):
    """Measured fp64 FMA throughput (TFLOP/s) of this GPU, from the library's
    DFMA probe; datasheet figure when the probe is unavailable."""
    try:
        from paper_1901_10559_b200 import _native

        lib = _native.load()
        v = float(lib.ids_probe_fp64_tflops(ctx.torch.cuda.current_stream().cuda_stream))
        if v > 0:
            return v, "measured (ids_probe_fp64_tflops: DFMA chains on every SM)"
    except Exception:
        pass
    return FP64_PEAK_DATASHEET, "datasheet"


def measure(ctx, wl, steps, warmup, args, headline):
    """Time one workload: trials (value), single-call latency, the dominant
    kernel alone (roofline), end to end from host buffers; CPU baseline and
    parity at N = 1 on rank 0."""
    torch = ctx.torch
    from paper_1901_10559_b200 import _native

    lib = _native.load()
    # single-call latency (one ID, nothing overlapped): the "ID seconds"
    for s in range(2):
        wl.single(s)
    ctx.barrier()
    t_single = []
    for s in range(3):
        t_single.append(ctx.events(lambda i, s=s: wl.single(100 + s), 1))
    single_ms = ctx.max_over_ranks(float(np.median(t_single)))

    # device-resident trials (value); warm-up sized to one timed batch
    wl.trials(range(max(warmup, steps)))
    torch.cuda.synchronize()
    clocks = busy0 = None
    if headline:
        clocks = Clocks(ctx.rank == 0)
        time.sleep(1.0)
        busy0 = time.time()
        while time.time() - busy0 < 1.0:
            wl.trials(range(steps))
        torch.cuda.synchronize()
    ctx.barrier()
    n0 = lib.ids_launch_count()
    ms = ctx.events(lambda i: wl.trials([1000 + s for s in range(steps)]), 1) / steps
    launches = (lib.ids_launch_count() - n0) // max(steps, 1)
    if getattr(wl, "graph", None) is not None:
        # graph replays launch the captured library kernels without host calls
        launches += wl.graph.launches
    ms = ctx.max_over_ranks(ms)
    clk = None
    if headline:
        busy1 = time.time()
        while time.time() - busy1 < 1.0:
            wl.trials(range(steps))
        torch.cuda.synchronize()
        clk = clocks.stop(torch.cuda.current_device(), window=(busy0, time.time()))

    # dominant kernel alone
    k_ms, k_bytes, extra = wl.kernel(max(3, steps))
    peak, peak_kind = peaks()
    achieved = k_bytes / (k_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic_of(wl.name, k_bytes),
            "kernel": wl.kernel_name, "peak_kind": peak_kind, "bytes_per_launch": k_bytes,
            "bytes_note": wl.bytes_note(), "kernel_ms": k_ms}
    if "flops_per_launch" in extra:
        fpk, fkind = fp64_peak(ctx)
        tf = extra["flops_per_launch"] / (k_ms * 1e-3) / 1e12
        roof["fp64"] = {"achieved": tf, "peak": fpk, "unit": "TFLOP/s", "frac": tf / fpk,
                        "peak_kind": fkind, "flops_per_launch": extra["flops_per_launch"]}
    if wl.name == "C3":
        # the streaming CSR kernel issues one fp64 L2 reduction per nonzero;
        # the measured scattered-RED peak (222 G/s, profiles/r01_l2_red_peak.txt)
        # is its real ceiling, reported beside the HBM roof
        nnz = int(wl.operand.nnz)
        red_ms = nnz / 222e9 * 1e3
        roof["ceiling"] = {"bound": "l2_fp64_reductions", "reductions_per_launch": int(nnz),
                           "peak_reductions_per_s": 222e9, "min_ms": red_ms,
                           "frac": red_ms / k_ms,
                           "note": "one fp64 L2 reduction per nonzero (RED.ADD.F64 into the "
                                   "L2-resident sketch)"}

    # end to end through the public API from host buffers
    e2e = None
    if not args.no_e2e:
        host, h2d = wl.host_copy()
        d = wl.e2e_call(host, 1)
        # second warm-up call: a repeated host-tensor shape is captured as a
        # CUDA graph on its second call (cp_tensor._host_graph_call); the
        # timed steps are the steady state, the H2D copies still in each
        wl.e2e_call(host, 2)
        ctx.barrier()
        reps = max(1, min(steps, 3))
        t0 = time.perf_counter()
        e_ms = ctx.max_over_ranks(ctx.events(lambda i: wl.e2e_call(host, 2000 + i), reps) / 1)
        res = d[0] if isinstance(d, tuple) else d
        d2h = int(res.coeffs.nbytes + res.cols.nbytes)
        e2e = {"value": wl.bytes_total / (e_ms * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(ctx.sum_over_ranks(h2d)),
               "d2h_bytes_per_step": d2h * ctx.world, "ms_per_step": e_ms,
               "wall_s": time.perf_counter() - t0}
        del host

    cpu = parity = None  # filled by cpu_legs() after every GPU timing

    out = {"value": wl.bytes_total / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
           "id_seconds": single_ms * 1e-3, "phases_ms": dict(
               {"sketch_kernel": k_ms}, **{k: v for k, v in extra.items() if k.endswith("ms")
                                           or "cpqr" in k or "hash" in k}),
           "roofline": roof, "cpu_baseline": cpu, "parity": parity, "e2e": e2e,
           "gpu_launches": int(launches), "config": config_of(wl.name, ctx.world, args.cpu_rows)}
    if clk is not None:
        out["clocks"] = clk
    return out


def cpu_legs(ctx, wls, results, args):
    """CPU baselines and parity, after every GPU timing of the run: the
    reference's BLAS / scipy threads stay busy for a while after they
    return, which would inflate the host-side launch times of anything
    timed next."""
    if ctx.world != 1 or args.no_cpu:
        return
    ref = RefCPU()
    for name, wl in wls.items():
        cpu, parity = wl.cpu_and_parity(ref, args.cpu_rows)
        results[name]["cpu_baseline"] = cpu
        results[name]["parity"] = parity


def traffic_of(name, nbytes):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    full capture (profiles/traffic.json), scaled to this rank's share."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        v = t.get(name)
        if v is None:
            return None
        full = t.get(name + "_bytes")
        return float(v) * (nbytes / full if full else 1.0)
    except Exception:
        return None


def main():
    args = parse()
    maybe_spawn(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

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
    ctx = Ctx(torch, dist, dev, rank, world)

    from paper_1901_10559_b200 import _native

    _native.load()
    wls, results = {}, {}
    wls[args.workload] = make_workload(ctx, args.workload)
    head = results[args.workload] = measure(ctx, wls[args.workload], args.steps, args.warmup, args,
                                            headline=True)
    secondary = None
    if not args.no_secondary:
        secondary = {}
        for name in ("C2", "C3", "C4", "C5"):
            if name == args.workload:
                continue
            wls[name] = make_workload(ctx, name)
            secondary[name] = results[name] = measure(ctx, wls[name], 20, 5, args, headline=False)
    cpu_legs(ctx, wls, results, args)
    del wls
    torch.cuda.empty_cache()

    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded, paper_1901_10559_b200.generators)",
            "config": head["config"], "id_seconds": head["id_seconds"],
            "trials": ("K trials (seeds) of the same input queued back to back, one host sync "
                       "at the end (matrices); N = 1: dense inputs draw each hash on a side "
                       "stream under the previous sketch, sparse inputs draw them in batches "
                       "(4 concurrent) ahead of the sketches; N > 1: draws split over the "
                       "ranks and broadcast"),
            "phases_ms": head["phases_ms"], "roofline": head["roofline"],
            "cpu_baseline": head["cpu_baseline"], "parity": head["parity"], "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"], "clocks": head.get("clocks"),
            "secondary_configs": secondary,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

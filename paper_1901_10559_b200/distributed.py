"""Multi-GPU CountSketch / TensorSketch ID (one process per GPU).

The reference is single-process (SPEC.md:490 makes distribution a non-goal);
this module adds the two partitionings SURVEY.md section 8(e) derives:

* matrices: A is split into contiguous row blocks; every rank draws the SAME
  global hash (it is a deterministic function of the seed), sketches its
  block with the global bucket/sign slice (row0 offset), then ONE
  all-reduce(SUM) of the small L x R sketch (1.6 MB for configs[1]) over
  NCCL/NVLink; the k-step pivoted QR + solve then run redundantly on every
  rank, so no broadcast of j / P is needed;
* CP tensors: the R rank-1 terms are split into column blocks; column r of
  the TensorSketch depends only on column r of each factor, so each rank
  sketches its block independently.  The ID then runs as a COLUMN-distributed
  truncated CPQR (``cpqr_columns_sharded``): per step one
  all-gather of 4-double pivot candidates into a device tensor, the pivot
  picked by a kernel, and one all-reduce of the L-double pivot column (the
  non-owners contribute -0.0), with no host synchronization; the L x R
  sketch (262 MB for configs[4]) is never gathered.  ``cpqr="gather"`` keeps
  the all-gather + redundant CPQR variant.  Trials of several seeds are
  queued with one host synchronization (``*_sharded_trials``).

``seed=None`` draws fresh entropy on the group's rank 0 and broadcasts it;
every broadcast names the source by its global rank, so subgroups work.

The arithmetic goes through a backend object so the partitioning and the
collectives can be exercised on CPU with gloo (tests/test_distributed_gloo.py,
whose backend is the CPU oracle); the product backend is ``DeviceBackend``.
"""

import numpy as np
import torch
import torch.distributed as dist


def row_block(n, world, rank):
    """Contiguous block [r0, r1) of n rows owned by `rank` of `world`."""
    return n * rank // world, n * (rank + 1) // world


class DeviceBackend:
    """sm_100a kernels through the C ABI (the product path)."""

    def matrix_sketch(self, a_local, row0, in_dim, sketch_dim, seed, surjective):
        from . import _device
        from ._inputs import DenseOperand, SparseOperand, matrix_operand
        from ._native import IDS_FLAG_ORDERED
        from .sketch import CountSketchOp

        if isinstance(a_local, (DenseOperand, SparseOperand)):
            operand = a_local
        else:
            operand = matrix_operand(a_local)
        op = CountSketchOp(in_dim, sketch_dim, seed=seed, surjective=surjective)
        y = _device.empty((operand.cols, sketch_dim), torch.float64)
        flag = _device.zeros(1, torch.int32)
        op.sketch_into(operand, y, row0=row0, accumulate=False, flags=IDS_FLAG_ORDERED,
                       nonfinite=flag)
        return y, flag, operand

    def cpqr_shard(self, y_local, col0, k):
        return DeviceCpqrShard(y_local, col0, k)

    def coeffs_from_factors(self, rtop, perm, k, ncols, rank_tol, numerical_rank):
        """P from the assembled truncated factorization (ids_id_coeffs_f64)."""
        from . import _device
        from ._native import call, query
        from .matrix_id import DeviceId

        rt = _device.to_device(np.ascontiguousarray(rtop), torch.float64)
        pm = _device.to_device(np.asarray(perm, dtype=np.int32))
        nr = _device.to_device(np.array([numerical_rank], dtype=np.int32))
        p = _device.empty((k, ncols), torch.float64)
        de = _device.empty(1, torch.int32)
        nbytes = query("ids_id_coeffs_workspace_bytes", k, ncols)
        ws = _device.workspace(nbytes)
        call("ids_id_coeffs_f64", _device.ptr(rt), _device.ptr(pm), k, ncols, float(rank_tol),
             _device.ptr(nr), _device.ptr(p), _device.ptr(de), _device.ptr(ws), nbytes,
             _device.stream_ptr())
        return DeviceId(pm[:k], p, nr, de, k).to_host("tensorsketch")

    def confirm_nonfinite(self, operand):
        from . import _device
        from ._native import call

        conf = _device.zeros(1, torch.int32)
        if operand.kind == "dense":
            call("ids_dense_has_nonfinite", _device.ptr(operand.t), operand.rows, operand.cols,
                 operand.ld, operand.layout, _device.ptr(conf), _device.stream_ptr())
        else:
            call("ids_values_has_nonfinite", _device.ptr(operand.data), operand.nnz,
                 _device.ptr(conf), _device.stream_ptr())
        return conf

    def tensor_sketch(self, factors_local, weights_local, mode_dims, sketch_dim, seed):
        from .sketch import TensorSketchOp

        op = TensorSketchOp(mode_dims, sketch_dim, seed=seed)
        return op.apply_device(factors_local, weights_local)

    def matrix_id(self, y, rows, cols, rank, rank_tol, method):
        from .matrix_id import device_matrix_id

        return device_matrix_id(y, rows, cols, rank, rank_tol).to_host(method)


def _world(group):
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def _global_rank(group, r):
    """Global rank of group-local rank r (dist.broadcast's src is global)."""
    return dist.get_global_rank(group, r) if group is not None else r


def _coll_device(group):
    """Device for collective buffers: CUDA under NCCL, host under gloo."""
    backend = dist.get_backend(group)
    if "nccl" in str(backend).lower() and torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _agreed_entropy(group):
    """Fresh OS entropy (seed=None, sketch.py:77) agreed on by every rank:
    group-local rank 0 draws, everyone receives it."""
    ent = np.random.SeedSequence().entropy % (2**63)
    world, _ = _world(group)
    if world == 1:
        return int(ent)
    t = torch.tensor([ent], dtype=torch.int64, device=_coll_device(group))
    dist.broadcast(t, src=_global_rank(group, 0), group=group)
    return int(t.item())


def countsketch_id_sharded(a_local, row0, in_dim, rank, sketch_dim=None, seed=None,
                           rank_tol=1e-12, surjective=True, group=None, backend=None):
    """countsketch_id of the global matrix whose rows [row0, row0 + rows) are
    `a_local` on this rank.  Every rank returns the same decomposition."""
    from .matrix_id import check_matrix_id_args

    backend = backend or DeviceBackend()
    world, _ = _world(group)
    cols = a_local.shape[1]

    class _Shape:
        shape = (in_dim, cols)

    sketch_dim = check_matrix_id_args(_Shape, rank, sketch_dim, "countsketch")
    if seed is None:
        # every rank must draw the same hash: agree on fresh entropy first
        seed = _agreed_entropy(group)
    y, flag, operand = backend.matrix_sketch(a_local, row0, in_dim, sketch_dim, seed, surjective)
    if world > 1:
        dist.all_reduce(y, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    if bool(flag.item()):
        conf = backend.confirm_nonfinite(operand)
        if world > 1:
            dist.all_reduce(conf, op=dist.ReduceOp.MAX, group=group)
        if bool(conf.item()):
            raise ValueError("a contains non-finite entries")
    return backend.matrix_id(y, sketch_dim, cols, rank, rank_tol, "countsketch")


def trial_sharded_operators(in_dim, out_dim, seeds, surjective=False, group=None, index=True):
    """CountSketchOps for a sequence of trials on every rank of `group`, each
    hash drawn by ONE rank: trial t by rank t % world, all of a rank's draws
    enqueued up front on side streams, then, trial by trial, one broadcast of
    the packed (bucket, sign, draw counters) buffer -- 5 bytes per row -- from
    its owner.  The Fisher-Yates resolution of a draw is a sequential chain
    that does not shrink with the row shard, so drawing every trial on every
    rank would cost each rank the whole job's draws; split, each rank pays
    for about K / world of them.  Every rank yields bit-identical operators."""
    from . import _device
    from ._native import load
    from .sketch import PIPELINE_GRID_CAP, CountSketchOp, _side_streams

    world, me = _world(group)
    seeds = list(seeds)
    mine = [t for t in range(len(seeds)) if t % world == me]
    dev = _device.device()
    main = torch.cuda.current_stream()
    sides = _side_streams(dev, max(1, min(len(mine), 4)))
    lib = load()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    cap = max(PIPELINE_GRID_CAP, sms // max(1, min(len(mine), 4)))
    drawn = {}
    for n, t in enumerate(mine):
        st = sides[n % len(sides)]
        lib.ids_set_hash_grid_cap(cap)
        try:
            with torch.cuda.stream(st):
                op = CountSketchOp(in_dim, out_dim, seed=seeds[t], surjective=surjective)
                buf = op.packed()
                ev = torch.cuda.Event()
                ev.record()
        finally:
            lib.ids_set_hash_grid_cap(0)
        drawn[t] = (buf, ev)
    nbytes = CountSketchOp._packed_layout(in_dim)[2]
    for t in range(len(seeds)):
        owner = t % world
        if owner == me:
            buf, ev = drawn.pop(t)
            main.wait_event(ev)
            buf.record_stream(main)
        else:
            buf = _device.empty(nbytes, torch.uint8)
        src = _global_rank(group, owner)
        dist.broadcast(buf, src=src, group=group)
        op = CountSketchOp._from_packed(buf, in_dim, out_dim, surjective)
        if index:
            op._bucket_index()
        yield op


def countsketch_id_sharded_trials(a_local, row0, in_dim, rank, sketch_dim=None, seeds=(0,),
                                  rank_tol=1e-12, surjective=True, group=None, **pipe):
    """countsketch_id_sharded for several seeds, fully queued on the device:
    hash, sketch, all-reduce and ID of every trial are enqueued back to back
    and the host synchronizes once at the end (non-finite input is checked
    then, for all trials at once).  Every rank returns the same list."""
    from . import _device
    from ._inputs import DenseOperand, SparseOperand, matrix_operand
    from ._native import IDS_FLAG_ORDERED
    from .matrix_id import check_matrix_id_args, device_matrix_id
    from .sketch import batched_operators, id_stream, pipelined_operators

    world, _ = _world(group)
    operand = a_local if isinstance(a_local, (DenseOperand, SparseOperand)) else \
        matrix_operand(a_local)
    cols = operand.cols

    class _Shape:
        shape = (in_dim, cols)

    L = check_matrix_id_args(_Shape, rank, sketch_dim, "countsketch")
    seeds = list(seeds)
    outs, flags = [], []
    main = torch.cuda.current_stream()
    side = id_stream() if pipe.pop("id_side", True) else main
    # one rank: each trial's hash is drawn on a side stream while the previous
    # trial sketches (sketch.pipelined_operators); several ranks: the trials'
    # hashes are split over the ranks and broadcast (trial_sharded_operators).
    # Each trial's ID runs on a high-priority stream beside the next sketch.
    from .sketch import CountSketchOp

    index = CountSketchOp.needs_index(operand, IDS_FLAG_ORDERED)
    # a sparse sketch is short next to its I-row hash draw: the draws run in
    # batches, several at a time, with nothing else on the GPU, and the
    # sketches after them (C3: 2.4-2.6 vs 3.6 ms per trial with the draws
    # under the sketches); dense sketches are long enough to hide the draws
    batched = pipe.pop("batched", isinstance(operand, SparseOperand))
    if world > 1:
        ops = trial_sharded_operators(in_dim, L, seeds, surjective, group, index=index)
    elif batched:
        ops = batched_operators(in_dim, L, seeds, surjective, index=index,
                                **{k: v for k, v in pipe.items() if k in ("streams", "grid_cap", "batch")})
    else:
        ops = pipelined_operators(in_dim, L, seeds, surjective, index=index, **pipe)
    for op in ops:
        y = torch.empty((cols, L), dtype=torch.float64, device=torch.cuda.current_device())
        flag = torch.zeros(1, dtype=torch.int32, device=y.device)
        op.sketch_into(operand, y, row0=row0, accumulate=False, flags=IDS_FLAG_ORDERED,
                       nonfinite=flag)
        if world > 1:
            dist.all_reduce(y, op=dist.ReduceOp.SUM, group=group)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            outs.append(device_matrix_id(y, L, cols, rank, rank_tol).packed())
        y.record_stream(side)
        outs[-1].record_stream(main)
        flags.append(flag)
    main.wait_stream(side)
    if flags:
        bad = torch.stack(flags).max()
        if world > 1:
            dist.all_reduce(bad, op=dist.ReduceOp.MAX, group=group)
        if bool(bad.item()):
            conf = DeviceBackend().confirm_nonfinite(operand)
            if world > 1:
                dist.all_reduce(conf, op=dist.ReduceOp.MAX, group=group)
            if bool(conf.item()):
                raise ValueError("a contains non-finite entries")
    packed = torch.stack(outs) if outs else None
    from .matrix_id import DeviceId

    # one pinned copy for all trials
    host = _device.to_host(packed) if packed is not None else []
    return [DeviceId.unpack(v, rank, cols, "countsketch", copy=False) for v in host]


def tensorsketch_id_sharded(x_local, col0, total_terms, all_weights, rank, sketch_dim=None,
                            seed=None, rank_tol=1e-12, group=None, backend=None,
                            cpqr="columns"):
    """tensorsketch_id with the R terms split into column blocks: this rank
    holds terms [col0, col0 + R_local) of the (normalized) CpTensor in
    x_local.  Returns the TensorIdResult-like tuple (cols, coeffs,
    new_weights, numerical_rank, rank_deficient), identical on all ranks."""
    from .cp_tensor import check_tensor_id_args

    backend = backend or DeviceBackend()
    world, me = _world(group)

    class _X:
        rank = total_terms
        total_entries = int(np.prod(x_local.mode_dims))

    sketch_dim = check_tensor_id_args(_X, rank, sketch_dim, "tensorsketch")
    if seed is None:
        seed = _agreed_entropy(group)
    y_local = backend.tensor_sketch(x_local.factors, x_local.weights, x_local.mode_dims,
                                    sketch_dim, seed)
    if world > 1 and cpqr == "columns":
        d = cpqr_columns_sharded(y_local, col0, total_terms, rank, rank_tol, group, backend)
        weights = np.asarray(all_weights, dtype=np.float64)
        return d, weights[d.cols] * d.coeffs.sum(axis=1)
    if world > 1:
        counts = [row_block(total_terms, world, r) for r in range(world)]
        sizes = [b - a for a, b in counts]
        width = max(sizes)
        pad = torch.zeros((width, sketch_dim), dtype=y_local.dtype, device=y_local.device)
        pad[: y_local.shape[0]] = y_local
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        y = torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0).contiguous()
    else:
        y = y_local
    d = backend.matrix_id(y, sketch_dim, total_terms, rank, rank_tol, "tensorsketch")
    weights = np.asarray(all_weights, dtype=np.float64)
    new_weights = weights[d.cols] * d.coeffs.sum(axis=1)
    return d, new_weights


def tensorsketch_id_sharded_trials(x_local, col0, total_terms, all_weights, rank,
                                   sketch_dim=None, seeds=(0,), rank_tol=1e-12, group=None):
    """tensorsketch_id_sharded for several seeds, fully queued on the device
    (the tensor twin of countsketch_id_sharded_trials): each trial's mode
    hashes, TensorSketch block and ID (single-GPU CPQR at one rank, the
    device-driven column-distributed CPQR beyond) are enqueued back to back
    and the host synchronizes once, on one packed copy of every trial's
    (j, P).  Returns [(InterpolativeDecomposition, new_weights)], identical
    on every rank and to separate tensorsketch_id calls."""
    from . import _device
    from .cp_tensor import check_tensor_id_args
    from .matrix_id import DeviceId, device_matrix_id
    from .sketch import TensorSketchOp

    world, me = _world(group)

    class _X:
        rank = total_terms
        total_entries = int(np.prod(x_local.mode_dims))

    L = check_tensor_id_args(_X, rank, sketch_dim, "tensorsketch")
    blocks = [row_block(total_terms, world, r) for r in range(world)]
    outs = []
    for s in seeds:
        y, nrm = TensorSketchOp(x_local.mode_dims, L, seed=s).apply_device(
            x_local.factors, x_local.weights, norms=True)
        if world == 1:
            d = device_matrix_id(y, L, total_terms, rank, rank_tol, colnorm2=nrm)
        else:
            d = _dcpqr_device(DeviceCpqrShard(y, col0, rank), blocks, total_terms, rank,
                              rank_tol, group)
        outs.append(d.packed())
    host = _device.to_host(torch.stack(outs)) if outs else []
    weights = np.asarray(all_weights, dtype=np.float64)
    res = []
    for v in host:
        d = DeviceId.unpack(v, rank, total_terms, "tensorsketch", copy=False)
        res.append((d, weights[d.cols] * d.coeffs.sum(axis=1)))
    return res


# ---- column-distributed truncated CPQR ---------------------
class DeviceCpqrShard:
    """This rank's column block of an L x R sketch for the column-distributed
    CPQR (ids_dcpqr_*): y is a CUDA (ncols, L) tensor, i.e. col-major L x
    ncols, holding global columns [col0, col0 + ncols)."""

    def __init__(self, y, col0, k):
        from . import _device
        from ._native import call, query

        self._d, self._call = _device, call
        self.y = y.contiguous()
        self.n, self.m = (int(v) for v in self.y.shape)
        self.col0, self.k = int(col0), int(k)
        self.nbytes = query("ids_dcpqr_workspace_bytes", self.m, self.n, self.k)
        self.ws = _device.workspace(self.nbytes)
        self.cand = _device.empty(4, torch.float64)
        self.a = _device.zeros(self.m, torch.float64)
        call("ids_dcpqr_init_f64", _device.ptr(self.y), self.m, self.n, self.m, self.k,
             self.col0, _device.ptr(self.cand), _device.ptr(self.ws), self.nbytes,
             _device.stream_ptr())

    def owns(self, col):
        return self.col0 <= col < self.col0 + self.n

    def pivot(self, kk, cs, ps, ck):
        d = self._d
        self._call("ids_dcpqr_pivot_f64", d.ptr(self.y), self.m, self.n, self.m, self.k,
                   self.col0, kk, cs, ps, ck, d.ptr(self.a), d.ptr(self.ws), self.nbytes,
                   d.stream_ptr())
        return self.a

    def step(self, kk, cs, a):
        d = self._d
        self._call("ids_dcpqr_step_f64", d.ptr(self.y), self.m, self.n, self.m, self.k,
                   self.col0, kk, cs, d.ptr(a), d.ptr(self.cand), d.ptr(self.ws), self.nbytes,
                   d.stream_ptr())

    # device-driven steps (ids_dcpqr_select / pivot_dev / step_dev): the pivot
    # never visits the host
    device_steps = True

    def select(self, cands, kk):
        """piv (device int64[3]) from the gathered candidates (device, shard order)."""
        d = self._d
        if not hasattr(self, "piv"):
            self.piv = d.empty(3, torch.int64)
        self._call("ids_dcpqr_select_f64", d.ptr(cands), int(cands.numel() // 4), kk,
                   d.ptr(self.piv), d.stream_ptr())
        return self.piv

    def pivot_dev(self, kk, piv):
        d = self._d
        self._call("ids_dcpqr_pivot_dev_f64", d.ptr(self.y), self.m, self.n, self.m, self.k,
                   self.col0, kk, d.ptr(piv), d.ptr(self.a), d.ptr(self.ws), self.nbytes,
                   d.stream_ptr())
        return self.a

    def step_dev(self, kk, piv, a):
        d = self._d
        self._call("ids_dcpqr_step_dev_f64", d.ptr(self.y), self.m, self.n, self.m, self.k,
                   self.col0, kk, d.ptr(piv), d.ptr(a), d.ptr(self.cand), d.ptr(self.ws),
                   self.nbytes, d.stream_ptr())

    def select_pivot(self, cands, kk):
        """select + pivot_dev in one launch; returns (piv, a)."""
        d = self._d
        if not hasattr(self, "piv"):
            self.piv = d.empty(3, torch.int64)
        self._call("ids_dcpqr_select_pivot_f64", d.ptr(self.y), self.m, self.n, self.m, self.k,
                   self.col0, kk, d.ptr(cands), int(cands.numel() // 4), d.ptr(self.piv),
                   d.ptr(self.a), d.ptr(self.ws), self.nbytes, d.stream_ptr())
        return self.piv, self.a

    def results(self):
        d = self._d
        pos = d.empty(max(self.n, 1), torch.int64)[: self.n]
        r = d.empty((self.k, max(self.n, 1)), torch.float64)[:, : self.n].contiguous()
        beta = d.empty(self.k, torch.float64)
        self._call("ids_dcpqr_results_f64", self.m, self.n, self.k, d.ptr(pos), d.ptr(r),
                   d.ptr(beta), d.ptr(self.ws), self.nbytes, d.stream_ptr())
        return pos, r, beta


def pick_pivot(cands, kk):
    """Global pivot from the per-shard candidates (rows: value, position,
    column, column at position kk) in shard order: largest value, ties to the
    lowest position (dgeqp3 / idamax); all-NaN norms keep position kk."""
    best, ck = None, -1
    for val, pos, col, nxt in np.asarray(cands, dtype=np.float64):
        if nxt >= 0:
            ck = int(nxt)
        if col < 0:
            continue
        if best is None or val > best[0] or (val == best[0] and pos < best[1]):
            best = (val, pos, col)
    if best is None:
        return ck, kk, ck
    return int(best[2]), int(best[1]), ck


def dcpqr_steps(shards, k, gather, broadcast):
    """Run the k steps over this process's shards.  gather(list of device
    cand tensors) -> host (S_total, 4) array in global shard order;
    broadcast(a_list, owner_col) makes every local shard's a equal to the
    owner's."""
    for kk in range(k):
        cs, ps, ck = pick_pivot(gather([sh.cand for sh in shards]), kk)
        a_list = [sh.pivot(kk, cs, ps, ck) for sh in shards]
        broadcast(a_list, cs)
        for sh, a in zip(shards, a_list):
            sh.step(kk, cs, a)


def assemble_pivoted(pos_all, r_all, beta, k, rank_tol):
    """perm (int64[R]), Rtop (k x R, pivoted order) and numerical_rank from
    the gathered per-column positions and R rows (global column order)."""
    pos_all = np.asarray(pos_all, dtype=np.int64)
    ncols = pos_all.size
    perm = np.empty(ncols, dtype=np.int64)
    perm[pos_all] = np.arange(ncols)
    rtop = np.zeros((k, ncols))
    r_all = np.asarray(r_all, dtype=np.float64)
    q = np.arange(k)[:, None]
    rtop[:, pos_all] = np.where(pos_all[None, :] >= q, r_all, 0.0)
    beta = np.asarray(beta, dtype=np.float64)
    lead = abs(beta[0])
    nr = int(np.sum(np.abs(beta) > rank_tol * lead)) if lead != 0.0 else 0
    return perm, rtop, nr


def _gather_blocks(pos, r, blocks, rank, group):
    """All-gather the per-rank positions and R rows (padded to the widest
    block) into global column order."""
    world = len(blocks)
    width = max(b1 - b0 for b0, b1 in blocks)
    pp = torch.zeros(width, dtype=torch.int64, device=pos.device)
    rp = torch.zeros((rank, width), dtype=torch.float64, device=r.device)
    pp[: pos.numel()] = pos
    rp[:, : r.shape[1]] = r
    pparts = [torch.empty_like(pp) for _ in range(world)]
    rparts = [torch.empty_like(rp) for _ in range(world)]
    dist.all_gather(pparts, pp, group=group)
    dist.all_gather(rparts, rp, group=group)
    sizes = [b1 - b0 for b0, b1 in blocks]
    pos = torch.cat([p[:s] for p, s in zip(pparts, sizes)])
    r = torch.cat([q[:, :s] for q, s in zip(rparts, sizes)], dim=1)
    return pos, r


def _dcpqr_device(shard, blocks, total_cols, rank, rank_tol, group):
    """The column-distributed CPQR driven entirely on the device: per step
    the candidates are gathered into a device tensor, the pivot is picked by
    a kernel (ids_dcpqr_select_f64) and the pivot column is summed over the
    ranks (the non-owners contribute -0.0, so the sum is the owner's column
    bit for bit); the factors are assembled and P solved on the device.  No
    host synchronization: returns a DeviceId (identical on every rank)."""
    from . import _device
    from ._native import call, query
    from .matrix_id import DeviceId

    world = len(blocks)
    nccl = world > 1 and "nccl" in str(dist.get_backend(group)).lower()
    gathered = torch.empty((world, 4), dtype=torch.float64, device=shard.cand.device)
    for kk in range(rank):
        c = shard.cand.reshape(1, 4)
        if nccl:
            dist.all_gather_into_tensor(gathered, c, group=group)
            c = gathered
        elif world > 1:
            parts = [torch.empty_like(c) for _ in range(world)]
            dist.all_gather(parts, c, group=group)
            c = torch.cat(parts)
        piv, a = shard.select_pivot(c, kk)  # one launch
        if world > 1:
            dist.all_reduce(a, op=dist.ReduceOp.SUM, group=group)
        shard.step_dev(kk, piv, a)
    pos, r, beta = shard.results()
    if world > 1:
        pos, r = _gather_blocks(pos, r, blocks, rank, group)
    # assemble_pivoted on the device: perm[pos] = column, Rtop[:, pos] = R
    # rows (upper trapezoid), numerical rank from the diagonal beta
    dev = pos.device
    perm = torch.empty(total_cols, dtype=torch.int32, device=dev)
    perm[pos] = torch.arange(total_cols, dtype=torch.int32, device=dev)
    q = torch.arange(rank, device=dev)[:, None]
    rtop = torch.zeros((rank, total_cols), dtype=torch.float64, device=dev)
    rtop[:, pos] = torch.where(pos[None, :] >= q, r, torch.zeros((), dtype=r.dtype, device=dev))
    lead = beta[0].abs()
    nr = torch.where(lead != 0, (beta.abs() > rank_tol * lead).sum(), 0).to(torch.int32)
    nr = nr.reshape(1)
    p = _device.empty((rank, total_cols), torch.float64)
    de = _device.empty(1, torch.int32)
    nbytes = query("ids_id_coeffs_workspace_bytes", rank, total_cols)
    ws = _device.workspace(nbytes)
    call("ids_id_coeffs_f64", _device.ptr(rtop), _device.ptr(perm), rank, total_cols,
         float(rank_tol), _device.ptr(nr), _device.ptr(p), _device.ptr(de), _device.ptr(ws),
         nbytes, _device.stream_ptr())
    return DeviceId(perm[:rank], p, nr, de, rank)


def cpqr_columns_sharded(y_local, col0, total_cols, rank, rank_tol=1e-12, group=None,
                         backend=None):
    """ID of an L x R sketch whose columns [col0, col0 + R_local) live on this
    rank (y_local: (R_local, L)), by the column-distributed truncated CPQR;
    the same InterpolativeDecomposition on every rank."""
    backend = backend or DeviceBackend()
    world, me = _world(group)
    blocks = [row_block(total_cols, world, r) for r in range(world)]
    if (col0, col0 + int(y_local.shape[0])) != blocks[me]:
        # the owner lookup and the all-gather sizes assume the row_block split
        raise ValueError(f"rank {me} holds columns [{col0}, {col0 + int(y_local.shape[0])}) "
                         f"but the split of {total_cols} over {world} ranks gives {blocks[me]}")
    shard = backend.cpqr_shard(y_local, col0, rank)

    def gather(cands):
        c = cands[0].reshape(1, 4)
        if world > 1:
            parts = [torch.empty_like(c) for _ in range(world)]
            dist.all_gather(parts, c, group=group)
            c = torch.cat(parts)
        return c.cpu().numpy()

    def broadcast(a_list, cs):
        if world > 1:
            owner = next(r for r, (b0, b1) in enumerate(blocks) if b0 <= cs < b1)
            dist.broadcast(a_list[0], src=_global_rank(group, owner), group=group)

    if getattr(shard, "device_steps", False):
        return _dcpqr_device(shard, blocks, total_cols, rank, rank_tol, group).to_host(
            "tensorsketch")
    dcpqr_steps([shard], rank, gather, broadcast)
    pos, r, beta = shard.results()
    if world > 1:
        pos, r = _gather_blocks(pos, r, blocks, rank, group)
    perm, rtop, nr = assemble_pivoted(pos.cpu().numpy(), r.cpu().numpy(), beta.cpu().numpy(),
                                      rank, rank_tol)
    return backend.coeffs_from_factors(rtop, perm, rank, total_cols, rank_tol, nr)

"""CountSketch and TensorSketch operators on B200.

Drop-in for reference ``pkg/src/idsketch/sketch.py:51-207``: same
constructors, attributes (``bucket`` int64, ``sign`` float64 +-1, ``in_dim``,
``out_dim``, ``surjective``; ``mode_ops``, ``seed``, ``mode_dims``),
``from_arrays``, ``apply``, ``materialize`` and the TensorSketch composite-hash
helpers.  The hash is drawn ON THE DEVICE (bit-exact with numpy's PCG64
stream, ``ids_countsketch_hash``) and kept there; ``bucket``/``sign`` are
host copies fetched on first access.  ``apply`` runs the sm_100a sketch
kernels; host inputs return numpy arrays, CUDA-tensor inputs return CUDA
tensors.
"""

import numpy as np
import scipy.sparse as sp
import torch

from . import _device
from ._inputs import DenseOperand, SparseOperand, matrix_operand
from ._native import IDS_ERETRY, IDS_FLAG_DETERMINISTIC, IDS_FLAG_ORDERED, call, load, query

_MAX_MATERIALIZE = 50_000_000  # sketch.py:30
# Up to this many nonzeros an ordered request keeps scipy's summation order
# (one bucket-gather pass per bucket: Y bit-identical).  Above it the CSR
# sketch streams A once and reduces into an L2-resident Y (equal to scipy's Y
# up to summation-order rounding, ~1e-16 relative), or -- under
# torch.use_deterministic_algorithms -- splits each bucket into row segments
# combined in a fixed order (run-to-run identical).
ORDERED_SPARSE_MAX_NNZ = 1 << 24
_SPARSE_MODES = ("auto", "ordered", "deterministic", "stream")
_sparse_mode = "auto"
_warned_stream = False


class NondeterministicSketchWarning(UserWarning):
    """The streaming CSR sketch sums each Y entry in L2 reductions whose
    order varies run to run (Y within ~1e-16 relative of scipy's)."""


def set_sparse_sketch_mode(mode):
    """Summation order of the CSR CountSketch (the reference's scipy S @ A is
    sequential and deterministic, sketch.py:116-122):

    * "auto" (default): scipy's order bit for bit up to ORDERED_SPARSE_MAX_NNZ
      nonzeros, the streaming kernel above (fast, not run-to-run identical;
      a NondeterministicSketchWarning is issued once), or fixed-order
      segments under torch.use_deterministic_algorithms(True);
    * "ordered": scipy's order at any size (bucket-gather kernel, slower);
    * "deterministic": fixed-order segments at any size (run-to-run identical);
    * "stream": the streaming kernel at any size (no warning).
    Returns the previous mode."""
    global _sparse_mode
    if mode not in _SPARSE_MODES:
        raise ValueError(f"mode must be one of {_SPARSE_MODES}, got {mode!r}")
    prev, _sparse_mode = _sparse_mode, mode
    return prev


def _sparse_flags(operand, flags):
    """CSR flags after the sparse sketch mode (see set_sparse_sketch_mode)."""
    global _warned_stream
    if _sparse_mode == "ordered":
        return (flags | IDS_FLAG_ORDERED) & ~IDS_FLAG_DETERMINISTIC
    if _sparse_mode == "deterministic":
        return (flags | IDS_FLAG_DETERMINISTIC) & ~IDS_FLAG_ORDERED
    if _sparse_mode == "stream":
        return flags & ~(IDS_FLAG_ORDERED | IDS_FLAG_DETERMINISTIC)
    if operand.nnz > ORDERED_SPARSE_MAX_NNZ and flags & IDS_FLAG_ORDERED:
        flags &= ~IDS_FLAG_ORDERED
    if torch.are_deterministic_algorithms_enabled():
        flags |= IDS_FLAG_DETERMINISTIC
    if not flags & (IDS_FLAG_ORDERED | IDS_FLAG_DETERMINISTIC) and not _warned_stream:
        import warnings

        _warned_stream = True
        warnings.warn(
            f"CSR input with {operand.nnz} nonzeros is sketched by the streaming kernel: Y "
            "matches scipy's to rounding but is not run-to-run identical; use "
            "set_sparse_sketch_mode('ordered' or 'deterministic') for a fixed order",
            NondeterministicSketchWarning, stacklevel=4)
    return flags


def _seed_entropy(seed):
    """sketch.py:33-39."""
    if seed is None:
        return np.random.SeedSequence().entropy
    if isinstance(seed, np.random.SeedSequence):
        return seed.entropy
    return int(seed)


def seed_state(seed):
    """The (state, inc) of the fresh PCG64 that ``np.random.default_rng(seed)``
    builds (sketch.py:77): SeedSequence hashing is numpy's own host code.  A
    Generator seed (default_rng returns it as is) starts at its current state
    (see _generator_state)."""
    if isinstance(seed, np.random.Generator):
        return _generator_state(seed)
    st = np.random.PCG64(seed).state["state"]
    return int(st["state"]), int(st["inc"])


def _generator_state(gen):
    """(state, inc) of a PCG64-backed Generator passed as seed.  The device
    draws start at a 64-bit boundary, so a pending 32-bit half (left by an
    odd number of earlier 32-bit draws) is not supported."""
    bg = gen.bit_generator
    if not isinstance(bg, np.random.PCG64):
        raise TypeError(f"Generator seeds must use PCG64 (numpy's default), got "
                        f"{type(bg).__name__}")
    st = bg.state
    if st["has_uint32"]:
        raise ValueError("Generator holds a pending 32-bit half-draw; draw an even number of "
                         "32-bit values first or pass an int / SeedSequence seed")
    return int(st["state"]["state"]), int(st["state"]["inc"])


def _advance_generator(gen, n32):
    """Leave `gen` where numpy's own draws of n32 32-bit values would: past
    ceil(n32 / 2) PCG64 outputs, the high half of the last one pending when
    n32 is odd."""
    bg = gen.bit_generator
    n64 = (int(n32) + 1) // 2
    if n64 == 0:
        return
    probe = np.random.PCG64()
    probe.state = bg.state
    probe.advance(n64 - 1)
    last = int(probe.random_raw())
    st = probe.state
    if n32 % 2:
        st["has_uint32"], st["uinteger"] = 1, last >> 32
    else:
        st["has_uint32"], st["uinteger"] = 0, 0
    bg.state = st


def _split(v):
    return (v >> 64) & 0xFFFFFFFFFFFFFFFF, v & 0xFFFFFFFFFFFFFFFF


def _check_rows(a, in_dim, kind):
    """sketch.py:42-48."""
    ndim = a.dim() if isinstance(a, torch.Tensor) else np.ndim(a)
    if ndim != 2:
        raise ValueError("sketch input must be 2-D")
    if a.shape[0] != in_dim:
        raise ValueError(f"{kind} expects {in_dim} input rows, got {a.shape[0]}")


class CountSketchOp:
    """Bucket-and-sign sketch S (reference sketch.py:51-125).

    In surjective mode the bucket map is a random permutation of
    [0..out_dim) followed by iid uniform values, so every output row receives
    at least one input row.
    """

    def __init__(self, in_dim, out_dim, seed=None, surjective=False, _seed_dev=None):
        if in_dim < 1 or out_dim < 1:
            raise ValueError("dimensions must be positive")
        if surjective and out_dim > in_dim:
            raise ValueError(
                f"surjective mode requires out_dim <= in_dim, got {out_dim} > {in_dim}"
            )
        self.in_dim = int(in_dim)
        self.out_dim = int(out_dim)
        self.surjective = bool(surjective)
        self._bucket_h = None
        self._sign_h = None
        self._index = None
        self._bucket_d = _device.empty(self.in_dim, torch.int32)
        self._sign_d = _device.empty(self.in_dim, torch.int8)
        self._draws = _device.empty(4, torch.int64)
        nbytes = query("ids_hash_workspace_bytes", self.in_dim, self.out_dim, int(self.surjective))
        ws = _device.workspace(nbytes)
        tail = (self.in_dim, self.out_dim, int(self.surjective), _device.ptr(self._bucket_d),
                _device.ptr(self._sign_d), _device.ptr(self._draws), _device.ptr(ws), nbytes,
                _device.stream_ptr())
        if _seed_dev is not None:
            # (state_hi, state_lo, inc_hi, inc_lo) read by the kernels from
            # device memory: the draw can be captured in a CUDA graph once and
            # replayed for any seed (cp_tensor.TensorIdGraph)
            call("ids_countsketch_hash_dev", _device.ptr(_seed_dev), *tail)
        else:
            state, inc = seed_state(seed)
            sh, sl = _split(state)
            ih, il = _split(inc)
            call("ids_countsketch_hash", sh, sl, ih, il, *tail)
        self._checked = False
        if isinstance(seed, np.random.Generator):
            # default_rng(gen) draws from gen itself (sketch.py:77): advance it
            _advance_generator(seed, sum(self.draws))

    @classmethod
    def from_arrays(cls, bucket, sign, out_dim=None):
        """Operator from explicit bucket and sign arrays (sketch.py:91-106)."""
        bucket = np.asarray(bucket, dtype=np.int64)
        sign = np.asarray(sign, dtype=np.float64)
        if bucket.ndim != 1 or bucket.shape != sign.shape:
            raise ValueError("bucket and sign must be 1-D arrays of equal length")
        if not np.isin(sign, (-1.0, 1.0)).all():
            raise ValueError("signs must be +-1")
        op = cls.__new__(cls)
        op.in_dim = bucket.size
        op.out_dim = int(bucket.max()) + 1 if out_dim is None else int(out_dim)
        op.surjective = bool(np.unique(bucket).size == op.out_dim)
        if bucket.size and (bucket.min() < 0 or bucket.max() >= op.out_dim):
            raise ValueError("bucket values must lie in [0, out_dim)")
        op._bucket_h = bucket
        op._sign_h = sign
        op._bucket_d = _device.to_device(bucket.astype(np.int32))
        op._sign_d = _device.to_device(sign.astype(np.int8))
        op._draws = None
        op._index = None
        op._checked = True
        return op

    # ---- packed form (one buffer per operator, for a collective) -----------
    @staticmethod
    def _packed_layout(in_dim):
        """Byte offsets of (bucket int32, sign int8, draws int64[4]) in the
        packed buffer, and its total size."""
        b1 = 4 * in_dim
        d0 = (b1 + in_dim + 15) // 16 * 16
        return b1, d0, d0 + 32

    def packed(self):
        """bucket, sign and the draw counters in one device uint8 buffer."""
        b1, d0, n = self._packed_layout(self.in_dim)
        buf = _device.empty(n, torch.uint8)
        buf[:b1].view(torch.int32).copy_(self._bucket_d)
        buf[b1:b1 + self.in_dim].view(torch.int8).copy_(self._sign_d)
        if self._draws is not None:
            buf[d0:].view(torch.int64).copy_(self._draws)
        else:
            buf[d0:].zero_()
        return buf

    @classmethod
    def _from_packed(cls, buf, in_dim, out_dim, surjective):
        """Operator over a packed buffer (views, no copy): the hash drawn by
        another rank and broadcast (distributed.countsketch_id_sharded_trials)."""
        b1, d0, n = cls._packed_layout(in_dim)
        op = cls.__new__(cls)
        op.in_dim, op.out_dim, op.surjective = int(in_dim), int(out_dim), bool(surjective)
        op._bucket_h = op._sign_h = op._index = None
        op._bucket_d = buf[:b1].view(torch.int32)
        op._sign_d = buf[b1:b1 + in_dim].view(torch.int8)
        op._draws = buf[d0:n].view(torch.int64)
        op._checked = False
        return op

    def record_stream(self, stream):
        """Mark the operator's device arrays as used on `stream` (they may have
        been drawn on another stream, see pipelined_operators)."""
        for t in (self._bucket_d, self._sign_d, self._draws):
            if t is not None:
                t.record_stream(stream)
        if self._index is not None:
            for t in self._index:
                t.record_stream(stream)
        for name in ("_plan", "_split_plan"):
            if getattr(self, name, None) is not None:
                getattr(self, name).record_stream(stream)

    # ---- host views -------------------------------------------------------
    def _check_draws(self):
        if self._checked or self._draws is None:
            return
        status = int(self._draws[3].item())
        if status == IDS_ERETRY:  # pragma: no cover - needs ~e^-100 luck
            raise RuntimeError("hash draw buffer exhausted; rebuild the operator")
        self._checked = True

    @property
    def bucket(self):
        if self._bucket_h is None:
            self._check_draws()
            self._bucket_h = _device.to_host(self._bucket_d).astype(np.int64)
        return self._bucket_h

    @property
    def sign(self):
        if self._sign_h is None:
            self._check_draws()
            self._sign_h = _device.to_host(self._sign_d).astype(np.float64)
        return self._sign_h

    @property
    def draws(self):
        """32-bit draws consumed by (phase A, permutation, signs)."""
        if self._draws is None:
            return None
        return tuple(int(v) for v in _device.to_host(self._draws)[:3])

    def materialize(self):
        """Dense L x I operator (sketch.py:124-125; test helper)."""
        out = np.zeros((self.out_dim, self.in_dim))
        out[self.bucket, np.arange(self.in_dim)] = self.sign
        return out

    # ---- device ------------------------------------------------------------
    def bucket_index(self):
        """(order_signed int32[I], bstart int64[L+1]) -- the CSR structure of S."""
        return self._bucket_index()[:2]

    def _bucket_index(self):
        """(order_signed, bstart, sorted_bucket) on the device."""
        if self._index is None:
            order = _device.empty(self.in_dim, torch.int32)
            bstart = _device.empty(self.out_dim + 1, torch.int64)
            keys = _device.empty(self.in_dim, torch.int32)
            nbytes = query("ids_bucket_index_workspace_bytes", self.in_dim, self.out_dim)
            ws = _device.workspace(nbytes)
            call(
                "ids_bucket_index", _device.ptr(self._bucket_d), _device.ptr(self._sign_d),
                self.in_dim, self.out_dim, _device.ptr(order), _device.ptr(bstart),
                _device.ptr(keys), _device.ptr(ws), nbytes, _device.stream_ptr(),
            )
            self._index = (order, bstart, keys)
        return self._index

    def _ts_plan(self):
        """Scatter plan of this operator as one TensorSketch mode (per-row
        bucket/sign code and rank within its bucket), built on the device
        once and cached (ids_ts_mode_plan)."""
        if getattr(self, "_plan", None) is None:
            order, bstart, keys = self._bucket_index()
            nbytes = query("ids_ts_mode_plan_bytes", self.in_dim)
            plan = _device.workspace(nbytes)
            call(
                "ids_ts_mode_plan", _device.ptr(order), _device.ptr(keys), _device.ptr(bstart),
                self.in_dim, self.out_dim, _device.ptr(plan), nbytes, _device.stream_ptr(),
            )
            self._plan = plan
        return self._plan

    def _ts_split_plan(self):
        """Folded scatter plan of this operator as one mode of the
        split-spectrum TensorSketch kernel (per-row slot b mod L/2, sign,
        b >= L/2, rank inside its chunk; per-chunk largest rank), built on
        the device from bucket / sign once and cached (ids_ts_split_plan)."""
        if getattr(self, "_split_plan", None) is None:
            nbytes = query("ids_ts_split_plan_bytes", self.in_dim, self.out_dim)
            plan = _device.workspace(nbytes)
            call(
                "ids_ts_split_plan", _device.ptr(self._bucket_d), _device.ptr(self._sign_d),
                self.in_dim, self.out_dim, _device.ptr(plan), nbytes, _device.stream_ptr(),
            )
            self._split_plan = plan
        return self._split_plan

    @staticmethod
    def needs_index(operand, flags=0):
        """Whether sketch_into(operand, flags=flags) reads the bucket index
        (dense kernels and the ordered / deterministic CSR kernels do; CSC
        and the streaming CSR kernel read bucket / sign directly)."""
        if isinstance(operand, DenseOperand):
            return True
        if operand.fmt == "csc":
            return False
        if _sparse_mode == "ordered" or _sparse_mode == "deterministic":
            return True
        if _sparse_mode == "stream":
            return False
        if operand.nnz > ORDERED_SPARSE_MAX_NNZ and flags & IDS_FLAG_ORDERED:
            flags &= ~IDS_FLAG_ORDERED
        if torch.are_deterministic_algorithms_enabled():
            flags |= IDS_FLAG_DETERMINISTIC
        return bool(flags & (IDS_FLAG_ORDERED | IDS_FLAG_DETERMINISTIC))

    def sketch_into(self, operand, y, row0=0, accumulate=False, flags=0, nonfinite=None):
        """Y (+)= S[:, row0:row0+rows] @ operand on the current stream.

        y: CUDA float64 tensor of shape (cols, out_dim) -- the col-major L x R
        sketch.  nonfinite: optional device int32[1] flag.
        """
        st = _device.stream_ptr()
        nf = _device.ptr(nonfinite)
        if isinstance(operand, DenseOperand):
            order, bstart = self.bucket_index()
            nbytes = query(
                "ids_countsketch_dense_workspace_bytes", operand.rows, operand.cols,
                self.out_dim, operand.layout,
            )
            ws = _device.workspace(nbytes)
            call(
                "ids_countsketch_dense_f64", _device.ptr(operand.t), operand.rows, operand.cols,
                operand.ld, operand.layout, row0, self.in_dim, _device.ptr(self._bucket_d),
                _device.ptr(self._sign_d), _device.ptr(order), _device.ptr(bstart),
                self.out_dim, _device.ptr(y), int(accumulate), int(flags), nf,
                _device.ptr(ws), nbytes, st,
            )
        elif isinstance(operand, SparseOperand) and operand.fmt == "csc":
            nbytes = query("ids_countsketch_csc_workspace_bytes", operand.cols, self.out_dim)
            ws = _device.workspace(nbytes)
            call(
                "ids_countsketch_csc_f64", _device.ptr(operand.indptr),
                int(operand.indptr.dtype == torch.int64), _device.ptr(operand.indices),
                _device.ptr(operand.data), operand.rows, operand.cols, operand.nnz, row0,
                self.in_dim, _device.ptr(self._bucket_d), _device.ptr(self._sign_d),
                self.out_dim, _device.ptr(y), int(accumulate), nf, _device.ptr(ws), nbytes, st,
            )
        elif isinstance(operand, SparseOperand):
            flags = _sparse_flags(operand, flags)
            if flags & (IDS_FLAG_ORDERED | IDS_FLAG_DETERMINISTIC):
                order, bstart = self.bucket_index()
            else:  # streaming pass: no bucket index needed
                order = bstart = None
            nbytes = query(
                "ids_countsketch_csr_workspace_bytes", operand.rows, operand.cols, operand.nnz,
                self.out_dim,
            )
            ws = _device.workspace(nbytes)
            call(
                "ids_countsketch_csr_f64", _device.ptr(operand.indptr),
                int(operand.indptr.dtype == torch.int64), _device.ptr(operand.indices),
                _device.ptr(operand.data), operand.rows, operand.cols, operand.nnz, row0,
                self.in_dim, _device.ptr(self._bucket_d), _device.ptr(self._sign_d),
                _device.ptr(order), _device.ptr(bstart), self.out_dim, _device.ptr(y),
                int(accumulate), int(flags), nf, _device.ptr(ws), nbytes, st,
            )
        else:  # pragma: no cover
            raise TypeError(f"unsupported operand {type(operand)!r}")

    def apply_device(self, a, flags=0, nonfinite=None):
        """S @ a as a CUDA tensor of shape (cols, out_dim) (col-major sketch)."""
        op = a if isinstance(a, (DenseOperand, SparseOperand)) else matrix_operand(a)
        if op.rows != self.in_dim:
            raise ValueError(f"CountSketch expects {self.in_dim} input rows, got {op.rows}")
        y = _device.empty((op.cols, self.out_dim), torch.float64)
        self.sketch_into(op, y, 0, False, flags, nonfinite)
        return y

    def apply(self, a):
        """Sketch `a` (sparse or dense, in_dim rows); returns a dense array
        (sketch.py:116-122).  CUDA-tensor input returns a CUDA tensor."""
        if not sp.issparse(a) and not isinstance(a, (DenseOperand, SparseOperand)):
            _check_rows(a, self.in_dim, "CountSketch")
        elif a.shape[0] != self.in_dim:
            raise ValueError(f"CountSketch expects {self.in_dim} input rows, got {a.shape[0]}")
        on_device = isinstance(a, torch.Tensor) and a.device.type == "cuda"
        if a.shape[1] == 0:
            return np.zeros((self.out_dim, 0))
        op = matrix_operand(a)
        y = self.apply_device(op, flags=IDS_FLAG_ORDERED).t()
        if on_device:
            return y
        return _device.to_host(y.contiguous())


class TensorSketchOp:
    """CountSketch whose hash and sign factor across tensor modes
    (reference sketch.py:128-207)."""

    def __init__(self, mode_dims, out_dim, seed=None, _seed_dev=None):
        mode_dims = [int(d) for d in mode_dims]
        if len(mode_dims) == 0:
            raise ValueError("need at least one mode")
        if any(d < 1 for d in mode_dims) or out_dim < 1:
            raise ValueError("dimensions must be positive")
        self.mode_dims = tuple(mode_dims)
        self.out_dim = int(out_dim)
        if _seed_dev is not None:  # device (N, 4) PCG64 states (see mode_seed_states)
            self.seed = None
            kw = [dict(_seed_dev=_seed_dev[n]) for n in range(len(mode_dims))]
        else:
            entropy = _seed_entropy(seed)
            self.seed = entropy
            kw = [dict(seed=np.random.SeedSequence([entropy, n])) for n in range(len(mode_dims))]
        self.mode_ops = _draw_modes(mode_dims, self.out_dim, kw)

    @staticmethod
    def mode_seed_states(n_modes, seed):
        """int64 (n_modes, 4) host array: the (state_hi, state_lo, inc_hi,
        inc_lo) words of mode n's PCG64, seeded SeedSequence([entropy, n])
        (reference sketch.py:143-150), as ids_countsketch_hash_dev reads them."""
        entropy = _seed_entropy(seed)
        out = np.empty((n_modes, 4), dtype=np.uint64)
        for n in range(n_modes):
            state, inc = seed_state(np.random.SeedSequence([entropy, n]))
            out[n] = (*_split(state), *_split(inc))
        return out.view(np.int64)

    @property
    def in_dim(self):
        return int(np.prod(self.mode_dims))

    def apply_device(self, factors, weights=None, norms=False):
        """Sketch of khatri_rao(factors) @ diag(weights) as a CUDA tensor of
        shape (ncols, out_dim) (col-major L x R); norms=True also returns the
        squared column norms of the sketch (device, or None)."""
        from .tensorsketch import tensorsketch_device

        return tensorsketch_device(self, factors, weights, norms=norms)

    def apply(self, factors, weights=None):
        """sketch.py:156-186: numpy L x R for host factors."""
        if len(factors) != len(self.mode_ops):
            raise ValueError(f"expected {len(self.mode_ops)} factors, got {len(factors)}")
        on_device = all(isinstance(f, torch.Tensor) and f.device.type == "cuda" for f in factors)
        y = self.apply_device(factors, weights).t()
        if on_device:
            return y
        return _device.to_host(y.contiguous())

    def composite_bucket(self):
        """Bucket of every Khatri-Rao row (last mode fastest), sketch.py:188-194."""
        total = np.zeros(1, dtype=np.int64)
        for op in self.mode_ops:
            total = (total[:, None] + op.bucket[None, :]).ravel()
        return total % self.out_dim

    def composite_sign(self):
        total = np.ones(1, dtype=np.float64)
        for op in self.mode_ops:
            total = (total[:, None] * op.sign[None, :]).ravel()
        return total

    def materialize(self):
        if self.in_dim * self.out_dim > _MAX_MATERIALIZE:
            raise ValueError("operator too large to materialize")
        dense = np.zeros((self.out_dim, self.in_dim))
        dense[self.composite_bucket(), np.arange(self.in_dim)] = self.composite_sign()
        return dense


_SIDE_STREAMS = {}
_MODE_STREAMS = {}


def _draw_modes(mode_dims, out_dim, kw):
    """The N per-mode CountSketchOps of a TensorSketchOp, each with its
    bucket index and (long modes) scatter plan, drawn CONCURRENTLY on side
    streams -- a dozen small kernels per mode that would otherwise run one
    after another -- joined back into the current stream (also inside a
    CUDA-graph capture, where they become parallel branches)."""
    from .tensorsketch import SCATTER_MIN_DIM, uses_split_kernel

    if len(mode_dims) == 1 or not torch.cuda.is_available():
        return [CountSketchOp(d, out_dim, **k) for d, k in zip(mode_dims, kw)]
    split = uses_split_kernel(len(mode_dims), out_dim)
    dev = _device.device()
    pool = _MODE_STREAMS.setdefault(dev.index, [])
    while len(pool) < len(mode_dims):
        pool.append(torch.cuda.Stream(device=dev))
    main = torch.cuda.current_stream()
    ops = []
    for d, k, st in zip(mode_dims, kw, pool):
        st.wait_stream(main)
        with torch.cuda.stream(st):
            op = CountSketchOp(d, out_dim, **k)
            if split:  # the split kernel reads its folded plan only
                op._ts_split_plan()
            else:
                op._bucket_index()
                if d >= SCATTER_MIN_DIM:
                    op._ts_plan()
        ops.append(op)
    for op, st in zip(ops, pool):
        main.wait_stream(st)
        op.record_stream(main)
    return ops
PIPELINE_DEPTH = 2     # draws in flight ahead of the trial being computed
PIPELINE_GRID_CAP = 16  # phase-B CTAs per background draw


def _side_streams(dev, n):
    pool = _SIDE_STREAMS.setdefault(dev.index, [])
    while len(pool) < n:
        pool.append(torch.cuda.Stream(device=dev))
    return pool[:n]


_ID_STREAMS = {}


def id_stream(dev=None):
    """High-priority side stream for the small per-trial ID (CPQR + P): its
    CTAs are dispatched as soon as any SM has room, so the ID of trial t runs
    beside the HBM-bound sketch of trial t + 1 instead of after it."""
    dev = dev or _device.device()
    st = _ID_STREAMS.get(dev.index)
    if st is None:
        lo, hi = torch.cuda.Stream.priority_range()
        st = _ID_STREAMS[dev.index] = torch.cuda.Stream(device=dev, priority=min(lo, hi))
    return st


BATCH_DRAW_STREAMS = 4    # concurrent draws in batched_operators
BATCH_DRAW_GRID_CAP = 74  # phase-B CTAs per concurrent draw
BATCH_DRAW_SIZE = 16      # operators drawn per batch


def batched_operators(in_dim, out_dim, seeds, surjective=False, index=True, streams=None,
                      grid_cap=None, batch=None):
    """CountSketchOps for a sequence of trials, drawn a batch at a time with
    nothing else running: each batch's draws go BATCH_DRAW_STREAMS at a time
    on side streams with a capped phase-B grid, the current stream joins
    them, then the batch's operators are yielded.  For operands whose sketch
    is short next to its hash draw (I = 1e7 CSR: 0.6 ms sketch, 2.5 ms
    draw), separating the phases beats drawing under the sketches:
    concurrent capped draws reach ~1.4 ms per draw
    (tools/exp_hash_concurrency.py) and the sketches run undisturbed."""
    seeds = list(seeds)
    if not seeds:
        return
    streams = BATCH_DRAW_STREAMS if streams is None else int(streams)
    grid_cap = BATCH_DRAW_GRID_CAP if grid_cap is None else int(grid_cap)
    batch = BATCH_DRAW_SIZE if batch is None else int(batch)
    dev = _device.device()
    main = torch.cuda.current_stream()
    sides = _side_streams(dev, max(streams, 1))
    lib = load()
    for b0 in range(0, len(seeds), batch):
        chunk = seeds[b0:b0 + batch]
        ops = []
        for st in sides:
            st.wait_stream(main)
        lib.ids_set_hash_grid_cap(grid_cap)
        try:
            for n, sd in enumerate(chunk):
                with torch.cuda.stream(sides[n % len(sides)]):
                    op = CountSketchOp(in_dim, out_dim, seed=sd, surjective=surjective)
                    if index:
                        op._bucket_index()
                ops.append(op)
        finally:
            lib.ids_set_hash_grid_cap(0)
        for st in sides:
            main.wait_stream(st)
        for op in ops:
            op.record_stream(main)
            yield op


def pipelined_operators(in_dim, out_dim, seeds, surjective=False, depth=None, grid_cap=None,
                        index=True):
    """CountSketchOps (hash + bucket index) for a sequence of trials, each
    drawn while earlier trials compute.

    A draw depends only on (in_dim, out_dim, seed, surjective), and its
    Fisher-Yates resolution is latency-bound.  Before yielding operator i
    (whose sketch the caller then enqueues on the current stream), the draws
    of operators up to i + depth are enqueued on side streams with their
    resolution grid capped (ids_set_hash_grid_cap), so they run beside the
    one-wave, HBM-bound sketch kernel instead of after it.  The current
    stream waits for each draw before its operator is used.  Measured on B200
    at configs[1] (I = 1e6, 10 trials, tools/exp_pipeline.py): 2.79 ms per
    trial at depth 2 / 16 CTAs, against 2.54 ms for the sketch + ID alone;
    depth 1 leaves the cooperative resolution waiting for room beside the
    sketch (3.6 ms), deeper pipelines add more concurrent draws than help.
    index=False skips the bucket index (operands whose sketch kernel reads
    bucket / sign directly: CSC, streaming CSR).
    """
    seeds = list(seeds)
    if not seeds:
        return
    depth = PIPELINE_DEPTH if depth is None else int(depth)
    grid_cap = PIPELINE_GRID_CAP if grid_cap is None else int(grid_cap)
    if depth == 0:  # no look-ahead: every draw in order on the current stream
        for sd in seeds:
            op = CountSketchOp(in_dim, out_dim, seed=sd, surjective=surjective)
            if index:
                op._bucket_index()
            yield op
        return
    dev = _device.device()
    main = torch.cuda.current_stream()
    sides = _side_streams(dev, max(depth, 1))
    lib = load()
    first = CountSketchOp(in_dim, out_dim, seed=seeds[0], surjective=surjective)
    if index:
        first._bucket_index()
    pending = [(first, None)]
    nxt = 1
    for i in range(len(seeds)):
        while nxt < len(seeds) and nxt <= i + depth:
            lib.ids_set_hash_grid_cap(grid_cap)
            try:
                with torch.cuda.stream(sides[nxt % len(sides)]):
                    op = CountSketchOp(in_dim, out_dim, seed=seeds[nxt], surjective=surjective)
                    if index:
                        op._bucket_index()
                    ev = torch.cuda.Event()
                    ev.record()
            finally:
                lib.ids_set_hash_grid_cap(0)
            pending.append((op, ev))
            nxt += 1
        op, ev = pending.pop(0)
        if ev is not None:
            main.wait_event(ev)
            op.record_stream(main)
        yield op
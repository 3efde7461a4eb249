"""Interpolative decomposition of matrices on B200.

Drop-in for reference ``pkg/src/idsketch/matrix_id.py``: ``countsketch_id``
(:170-182), ``matrix_sketch`` (:144-159), ``matrix_id`` (:87-113),
``check_matrix_id_args`` (:116-141) and ``InterpolativeDecomposition``
(:23-53), with the same signatures, defaults, return layout (``cols`` int32
j, ``coeffs`` float64 P of shape (k, cols) with an exact identity at
``cols``) and exceptions.  The whole pipeline -- hash draw, sketch, k-step
pivoted QR, triangular solve, identity scatter -- runs on the device; only
j and P cross back to the host.
"""

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from . import _device
from ._inputs import DenseOperand, SparseOperand, matrix_operand
from ._native import IDS_FLAG_ORDERED, call, query
from .linalg import DEFAULT_RANK_TOL, _check_finite_device, _col_major_device, device_cpqr
from .errors import SingularTriangleError
from .sketch import CountSketchOp

MATRIX_METHODS = ("deterministic", "countsketch")
DEFAULT_OVERSAMPLE = 10  # matrix_id.py:20


@dataclass(frozen=True)
class InterpolativeDecomposition:
    """Rank-k column ID: coeffs (k, cols) with an exact identity in the
    columns listed by `cols` (matrix_id.py:23-53)."""

    coeffs: np.ndarray
    cols: np.ndarray
    rank: int
    method: str
    numerical_rank: int
    rank_deficient: bool

    def reconstruct(self, a):
        """Dense rank-k approximation A[:, cols] @ coeffs of `a`."""
        sel = a[:, self.cols]
        out = sel @ self.coeffs
        if sp.issparse(out):
            out = out.toarray()
        return np.asarray(out)

    def to_dict(self):
        """JSON-ready form; column indices are 0-based."""
        return {
            "method": self.method,
            "k": int(self.rank),
            "j": [int(c) for c in self.cols],
            "p": self.coeffs.tolist(),
            "numerical_rank": int(self.numerical_rank),
            "rank_deficient": bool(self.rank_deficient),
        }


@dataclass
class DeviceId:
    """Device-resident ID of a sketch (results stay on the GPU until fetched)."""

    cols: torch.Tensor  # int32[k] view of perm
    coeffs: torch.Tensor  # float64[k, n]
    numerical_rank: torch.Tensor  # int32[1]
    deficient: torch.Tensor  # int32[1]
    rank: int

    def to_host(self, method, flag=None):
        """The decomposition on the host: one packed device->host copy.  With
        flag (device int32[1], e.g. the sketch's non-finite flag) returns
        (decomposition, bool(flag)) from the same copy."""
        vec = _device.to_host(self.packed(flag))
        d = self.unpack(vec[1:] if flag is not None else vec, self.rank,
                        self.coeffs.shape[1], method, copy=False)
        return (d, bool(vec[0])) if flag is not None else d

    def packed(self, flag=None):
        """cols, numerical_rank, deficient and coeffs packed in one float64
        device vector (indices are exact in float64), for one batched copy;
        flag (device int32[1]) is prepended when given."""
        parts = [self.cols.to(torch.float64), self.numerical_rank.to(torch.float64),
                 self.deficient.to(torch.float64), self.coeffs.reshape(-1)]
        if flag is not None:
            parts.insert(0, flag.to(torch.float64).reshape(1))
        return torch.cat(parts)

    @staticmethod
    def unpack(vec, rank, ncols, method, copy=True):
        """copy=False: coeffs is a view of vec -- for a vec that nobody
        reuses (a fresh to_host buffer), which the view then keeps alive;
        copying 1.6 MB of coefficients into fresh pages costs ~0.6 ms per
        result on the host (C3), more than the whole ID on the GPU."""
        cols = vec[:rank].astype(np.int32)
        nr, flags = int(vec[rank]), int(vec[rank + 1])
        if flags & 2:  # an exactly zero R11 diagonal reached the solve
            raise SingularTriangleError(f"zero diagonal entry at index {flags >> 2}")
        de = bool(flags & 1)
        coeffs = vec[rank + 2:rank + 2 + rank * ncols].reshape(rank, ncols)
        if copy:
            coeffs = coeffs.copy()
        return InterpolativeDecomposition(coeffs=coeffs, cols=cols, rank=rank, method=method,
                                          numerical_rank=nr, rank_deficient=de)


def device_matrix_id(y_cm, rows, cols, rank, rank_tol=DEFAULT_RANK_TOL, ld=None, colnorm2=None):
    """ID of the col-major rows x cols sketch in y_cm, on the device
    (matrix_id.py:87-113 via cpqr + _coeffs_from_pivoted).  colnorm2:
    optional device squared column norms of the sketch (see device_cpqr)."""
    f = device_cpqr(y_cm, rows, cols, rank, rank_tol, want_q=False, ld=ld, colnorm2=colnorm2)
    p = _device.empty((rank, cols), torch.float64)
    de = _device.empty(1, torch.int32)
    nbytes = query("ids_id_coeffs_workspace_bytes", rank, cols)
    ws = _device.workspace(nbytes)
    call(
        "ids_id_coeffs_f64", _device.ptr(f.rtop), _device.ptr(f.perm), rank, cols,
        float(rank_tol), _device.ptr(f.numerical_rank), _device.ptr(p), _device.ptr(de),
        _device.ptr(ws), nbytes, _device.stream_ptr(),
    )
    return DeviceId(f.perm[:rank], p, f.numerical_rank, de, rank)


def matrix_id(a, rank, rank_tol=DEFAULT_RANK_TOL):
    """Deterministic rank-`rank` ID of a dense matrix via column-pivoted QR."""
    t, rows, cols, ld = _col_major_device(a)
    _check_finite_device(t)
    if not 1 <= rank <= min(rows, cols):
        raise ValueError(f"rank must be in [1, {min(rows, cols)}], got {rank}")
    return device_matrix_id(t, rows, cols, rank, rank_tol, ld=ld).to_host("deterministic")


def check_matrix_id_args(a, rank, sketch_dim, method="countsketch"):
    """matrix_id.py:116-141: returns sketch_dim (default rank + 10)."""
    rows, ncols = a.shape
    if not 1 <= rank <= ncols:
        raise ValueError(f"rank must be in [1, {ncols}], got {rank}")
    if method == "deterministic":
        if rank > min(rows, ncols):
            raise ValueError(f"rank must be <= {min(rows, ncols)}, got {rank}")
        return None
    if sketch_dim is None:
        sketch_dim = rank + DEFAULT_OVERSAMPLE
    if sketch_dim < rank:
        raise ValueError(f"sketch dimension {sketch_dim} is below the target rank {rank}")
    if sketch_dim >= rows:
        raise ValueError(
            f"sketch dimension {sketch_dim} must be < {rows} input rows; "
            "use matrix_id directly instead"
        )
    return sketch_dim


def _method_op(rows, method, sketch_dim, seed, surjective):
    if method == "countsketch":
        return CountSketchOp(rows, sketch_dim, seed=seed, surjective=surjective)
    if method in ("gaussian", "srft"):
        raise NotImplementedError(
            f"{method!r} sketches are reference baselines outside this B200 hot path"
        )
    raise ValueError(f"unknown sketch method {method!r}")


def matrix_sketch(a, method, sketch_dim, seed=None, surjective=True):
    """Row sketch of `a` (matrix_id.py:144-159); dense numpy (L, cols)."""
    op = _method_op(a.shape[0], method, sketch_dim, seed, surjective)
    return op.apply(a)


def _raise_if_nonfinite(flag, operand):
    if not bool(flag.item()):
        return
    # Y had a NaN/Inf: confirm on the input itself (Y can also overflow)
    conf = _device.zeros(1, torch.int32)
    if isinstance(operand, DenseOperand):
        call(
            "ids_dense_has_nonfinite", _device.ptr(operand.t), operand.rows, operand.cols,
            operand.ld, operand.layout, _device.ptr(conf), _device.stream_ptr(),
        )
    else:
        call(
            "ids_values_has_nonfinite", _device.ptr(operand.data), operand.nnz,
            _device.ptr(conf), _device.stream_ptr(),
        )
    if bool(conf.item()):
        raise ValueError("a contains non-finite entries")


class _Shape:
    """Shape-only stand-in for check_matrix_id_args on host inputs."""

    def __init__(self, a):
        self.shape = tuple(a.shape) if sp.issparse(a) else tuple(np.shape(a))


def _host_input(a):
    """numpy / scipy / CPU-tensor A, 2-D and non-empty, that still has to be
    uploaded (anything else takes the plain path and its error order)."""
    if isinstance(a, (DenseOperand, SparseOperand)):
        return False
    if isinstance(a, torch.Tensor) and a.device.type == "cuda":
        return False
    try:
        shape = _Shape(a).shape
    except Exception:
        return False
    return len(shape) == 2 and shape[0] >= 1 and shape[1] >= 1


_UPLOAD_SIDE = {}


def _upload_side_stream():
    dev = _device.device()
    if dev.index not in _UPLOAD_SIDE:
        _UPLOAD_SIDE[dev.index] = torch.cuda.Stream(device=dev)
    return _UPLOAD_SIDE[dev.index]


def countsketch_device(a, rank, sketch_dim=None, seed=None, rank_tol=DEFAULT_RANK_TOL,
                       surjective=True, flags=IDS_FLAG_ORDERED, check_finite=True,
                       defer_check=False):
    """The device half of countsketch_id: returns (DeviceId, sketch (cols, L)).
    defer_check=True leaves the non-finite flag of the sketch on the device
    (DeviceId.nonfinite, DeviceId.operand) for the caller to read with the
    result -- no host synchronization before the ID is enqueued."""
    if _host_input(a):
        # host A: the hash is drawn on a side stream while A is uploaded (it
        # does not read A), then joined back into the current stream
        sketch_dim = check_matrix_id_args(_Shape(a), rank, sketch_dim, "countsketch")
        main, side = torch.cuda.current_stream(), _upload_side_stream()
        side.wait_stream(main)
        with torch.cuda.stream(side):
            op = CountSketchOp(_Shape(a).shape[0], sketch_dim, seed=seed, surjective=surjective)
        operand = matrix_operand(a)
        main.wait_stream(side)
        op.record_stream(main)
    else:
        operand = a if isinstance(a, (DenseOperand, SparseOperand)) else matrix_operand(a)
        sketch_dim = check_matrix_id_args(operand, rank, sketch_dim, "countsketch")
        op = CountSketchOp(operand.rows, sketch_dim, seed=seed, surjective=surjective)
    nonfinite = _device.zeros(1, torch.int32) if check_finite else None
    y = op.apply_device(operand, flags=flags, nonfinite=nonfinite)
    if check_finite and not defer_check:
        _raise_if_nonfinite(nonfinite, operand)
    d = device_matrix_id(y, sketch_dim, operand.cols, rank, rank_tol)
    if defer_check:
        d.nonfinite, d.operand = nonfinite, operand
    return d, y


def countsketch_id_trials(a, rank, sketch_dim=None, seeds=(0,), rank_tol=DEFAULT_RANK_TOL,
                          surjective=True):
    """countsketch_id of one matrix for several seeds (the paper averages 10
    trials).  A is uploaded once and nothing waits on the host until every
    trial is queued.  Returns a list of InterpolativeDecomposition, identical
    to separate countsketch_id calls."""
    from .distributed import countsketch_id_sharded_trials

    operand = a if isinstance(a, (DenseOperand, SparseOperand)) else matrix_operand(a)
    return countsketch_id_sharded_trials(operand, 0, operand.rows, rank, sketch_dim, seeds,
                                         rank_tol, surjective)


def countsketch_id(a, rank, sketch_dim=None, seed=None, rank_tol=DEFAULT_RANK_TOL, surjective=True):
    """Randomized ID from a CountSketch of the rows of `a` (matrix_id.py:170-182).

    The sketch costs one pass over A on the GPU; the ID of the
    (sketch_dim, cols) sketch then selects the columns.  Surjective bucket
    maps (the default) keep the sketch operator full rank.  Default
    sketch_dim is rank + 10.
    """
    d, _ = countsketch_device(a, rank, sketch_dim, seed, rank_tol, surjective, defer_check=True)
    out, bad = d.to_host("countsketch", flag=d.nonfinite)
    if bad:  # Y had a NaN / Inf: confirm on A itself (raises ValueError)
        _raise_if_nonfinite(d.nonfinite, d.operand)
    return out


__all__ = [
    "DEFAULT_OVERSAMPLE",
    "InterpolativeDecomposition",
    "MATRIX_METHODS",
    "check_matrix_id_args",
    "countsketch_device",
    "countsketch_id",
    "countsketch_id_trials",
    "device_matrix_id",
    "matrix_id",
    "matrix_sketch",
]

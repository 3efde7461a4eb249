"""Factorization kernels on the device: truncated CPQR and triangular solves.

Drop-in for reference ``pkg/src/idsketch/linalg.py:15-147`` (the parts on the
ID hot path): ``DEFAULT_RANK_TOL``, ``SingularTriangleError``, ``PivotedQr``,
``cpqr``, ``triangular_solve`` and the ``as_dense`` validator.  ``cpqr`` runs
``ids_cpqr_trunc_f64`` (k pivot steps of dgeqp3's rule) instead of a full
LAPACK factorization; ``perm`` therefore lists the k pivots first and the
remaining columns in the kernel's swap order (the reference returns LAPACK's
full pivot order -- identical first k entries, and the same column SET after
them, which is all the ID consumes).
"""

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from . import _device
from ._inputs import dense_operand
from ._native import IDS_COL_MAJOR, call, query
from .errors import SingularTriangleError

DEFAULT_RANK_TOL = 1e-12  # linalg.py:15

__all__ = [
    "DEFAULT_RANK_TOL",
    "PivotedQr",
    "SingularTriangleError",
    "as_dense",
    "cpqr",
    "device_cpqr",
    "is_sparse",
    "triangular_solve",
]


def as_dense(a, name="a"):
    """linalg.py:22-36: float64 F-ordered copy with shape/finiteness checks."""
    if sp.issparse(a):
        raise ValueError(f"{name} must be dense; densify sparse input explicitly")
    out = np.asfortranarray(a, dtype=np.float64)
    if out.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got ndim={out.ndim}")
    if out.size == 0:
        raise ValueError(f"{name} must be nonempty")
    if not np.isfinite(out).all():
        raise ValueError(f"{name} contains non-finite entries")
    return out


def is_sparse(a):
    return sp.issparse(a)


@dataclass(frozen=True)
class PivotedQr:
    """Rank-`k` partial column-pivoted QR (linalg.py:60-73)."""

    q: np.ndarray
    r: np.ndarray
    perm: np.ndarray
    numerical_rank: int


@dataclass
class DeviceQr:
    """Device-resident truncated CPQR of a col-major (cols, rows) sketch."""

    perm: torch.Tensor  # int32[cols]
    rtop: torch.Tensor  # float64[k, cols] (row-major)
    numerical_rank: torch.Tensor  # int32[1]
    q: torch.Tensor = None  # float64[k, rows] (col-major rows x k) or None


def device_cpqr(y_cm, rows, cols, rank, rank_tol=DEFAULT_RANK_TOL, want_q=False, ld=None,
                colnorm2=None):
    """Truncated CPQR of the col-major rows x cols matrix stored in y_cm
    (CUDA float64, column j at y_cm[j*ld : j*ld + rows]).  colnorm2: optional
    device ||Y[:, j]||^2 (the TensorSketch epilogue's), replacing the
    factorization's own initial norm pass."""
    ld = rows if ld is None else ld
    perm = _device.empty(cols, torch.int32)
    rtop = _device.empty((rank, cols), torch.float64)
    nr = _device.empty(1, torch.int32)
    q = _device.empty((rank, rows), torch.float64) if want_q else None
    nbytes = query("ids_cpqr_workspace_bytes", rows, cols, rank)
    ws = _device.workspace(nbytes)
    call(
        "ids_cpqr_trunc_norms_f64", _device.ptr(y_cm), rows, cols, ld, rank, float(rank_tol),
        _device.ptr(colnorm2), _device.ptr(perm), _device.ptr(rtop), _device.ptr(q),
        _device.ptr(nr), _device.ptr(ws), nbytes, _device.stream_ptr(),
    )
    return DeviceQr(perm, rtop, nr, q)


def _col_major_device(a):
    """Validated dense matrix -> (col-major CUDA tensor view, rows, cols, ld)."""
    op = dense_operand(a)
    t = op.t
    if op.layout != IDS_COL_MAJOR:
        t = t.t().contiguous()  # (cols, rows) contiguous == col-major rows x cols
        ld = op.rows
    else:
        t = t.t()  # (cols, rows) view with row stride ld
        ld = op.ld
    return t, op.rows, op.cols, ld


def _check_finite_device(t):
    if not bool(torch.isfinite(t).all().item()):
        raise ValueError("a contains non-finite entries")


def cpqr(a, rank, rank_tol=DEFAULT_RANK_TOL):
    """Column-pivoted Householder QR truncated to `rank` pivots (linalg.py:76-103).

    Pivoting selects the remaining column of largest (partial) norm, ties to
    the lowest column position, so |diag(r)| is nonincreasing.
    """
    t, rows, cols, ld = _col_major_device(a)
    _check_finite_device(t)
    if not 1 <= rank <= min(rows, cols):
        raise ValueError(f"rank must be in [1, {min(rows, cols)}], got {rank}")
    f = device_cpqr(t, rows, cols, rank, rank_tol, want_q=True, ld=ld)
    q = _device.to_host(f.q.t().contiguous())
    r = _device.to_host(f.rtop)
    perm = _device.to_host(f.perm)
    return PivotedQr(q=q, r=r, perm=perm, numerical_rank=int(_device.to_host(f.numerical_rank)[0]))


def triangular_solve(r, b, lower=False):
    """Solve r @ x = b for a nonsingular triangular `r` (linalg.py:130-147).

    Raises SingularTriangleError naming the first zero diagonal index.
    """
    r = np.asarray(r, dtype=np.float64)
    if r.ndim != 2 or r.shape[0] != r.shape[1]:
        raise ValueError(f"triangle must be square, got shape {r.shape}")
    b = np.asarray(b, dtype=np.float64)
    if b.shape[0] != r.shape[0]:
        raise ValueError(f"dimension mismatch: {r.shape} vs {b.shape}")
    diag = np.abs(np.diag(r))
    if (diag == 0.0).any():
        idx = int(np.argmin(diag != 0.0))
        raise SingularTriangleError(f"zero diagonal entry at index {idx}")
    if b.size == 0:
        return np.zeros_like(b)
    n = r.shape[0]
    b2 = b.reshape(n, -1)
    rd = _device.to_device(np.ascontiguousarray(r))
    bd = _device.to_device(np.ascontiguousarray(b2))
    xd = torch.empty_like(bd)
    bad = np.zeros(1, dtype=np.int64)
    call(
        "ids_triangular_solve_f64", _device.ptr(rd), _device.ptr(bd), n, b2.shape[1],
        int(bool(lower)), _device.ptr(xd), bad.ctypes.data, _device.stream_ptr(),
    )
    return _device.to_host(xd).reshape(b.shape)

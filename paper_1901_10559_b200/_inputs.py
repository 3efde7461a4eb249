"""Canonicalize user matrices into device-resident operands.

Mirrors the container rules of reference linalg.py:22-53 (as_dense /
as_csc): dense input must be a non-empty 2-D array and is read as float64;
sparse input is any scipy sparse container.  Instead of copying dense A into
Fortran order (linalg.py:29) the layout is kept: C-ordered A is sketched by
the row-major kernel, F-ordered A by the column-major one.  CSR and CSC are
native device formats; other scipy formats are converted to CSR first.
Finiteness (linalg.py:34, :51) is checked on the device, fused into the
sketch (see CountSketchOp._apply_dev).
"""

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp
import torch

from . import _device
from ._native import IDS_COL_MAJOR, IDS_ROW_MAJOR


@dataclass
class DenseOperand:
    t: torch.Tensor  # CUDA tensor holding the data (2-D view)
    rows: int
    cols: int
    layout: int
    ld: int
    host: bool  # came from host memory (results go back as numpy)

    @property
    def kind(self):
        return "dense"

    @property
    def shape(self):
        return (self.rows, self.cols)


@dataclass
class SparseOperand:
    fmt: str  # "csr" or "csc"
    indptr: torch.Tensor
    indices: torch.Tensor
    data: torch.Tensor
    rows: int
    cols: int
    nnz: int
    host: bool = True

    @property
    def kind(self):
        return self.fmt

    @property
    def shape(self):
        return (self.rows, self.cols)


def _dense_from_tensor(t, host):
    if t.dim() != 2:
        raise ValueError(f"a must be 2-D, got ndim={t.dim()}")
    if t.numel() == 0:
        raise ValueError("a must be nonempty")
    if t.dtype != torch.float64:
        t = t.to(torch.float64)
    rows, cols = t.shape
    if t.is_contiguous():
        layout, ld = IDS_ROW_MAJOR, max(cols, 1)
    elif t.t().is_contiguous():
        layout, ld = IDS_COL_MAJOR, max(rows, 1)
    elif t.stride(1) == 1 and t.stride(0) >= cols:
        layout, ld = IDS_ROW_MAJOR, t.stride(0)
    elif t.stride(0) == 1 and t.stride(1) >= rows:
        layout, ld = IDS_COL_MAJOR, t.stride(1)
    else:
        t = t.contiguous()
        layout, ld = IDS_ROW_MAJOR, cols
    if t.device.type != "cuda":
        if layout == IDS_ROW_MAJOR and ld != cols:
            t = t.contiguous()
            ld = cols
        if layout == IDS_COL_MAJOR and ld != rows:
            t = t.t().contiguous().t()
            ld = rows
        t = t.to(_device.device(), non_blocking=t.is_pinned())
        host = True
    return DenseOperand(t, rows, cols, layout, ld, host)


def dense_operand(a, name="a"):
    """Dense matrix -> DenseOperand (raises ValueError like as_dense)."""
    if sp.issparse(a):
        raise ValueError(f"{name} must be dense; densify sparse input explicitly")
    if isinstance(a, torch.Tensor):
        return _dense_from_tensor(a, host=a.device.type != "cuda")
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got ndim={arr.ndim}")
    if arr.size == 0:
        raise ValueError(f"{name} must be nonempty")
    if not (arr.flags.c_contiguous or arr.flags.f_contiguous):
        arr = np.ascontiguousarray(arr)
    if arr.flags.c_contiguous:
        t = torch.from_numpy(arr)
    else:
        t = torch.from_numpy(arr.T).t()
    return _dense_from_tensor(t, host=True)


def sparse_operand(a):
    """scipy sparse -> SparseOperand in CSR or CSC (device arrays)."""
    if a.format == "csc":
        fmt, m = "csc", a
    else:
        fmt, m = "csr", (a if a.format == "csr" else sp.csr_array(a))
    data = np.asarray(m.data, dtype=np.float64)
    indices = np.asarray(m.indices)
    if indices.dtype != np.int32:
        indices = indices.astype(np.int32)
    indptr = np.asarray(m.indptr)
    if indptr.dtype not in (np.int32, np.int64):
        indptr = indptr.astype(np.int64)
    dev = _device.device()
    rows, cols = m.shape
    return SparseOperand(
        fmt,
        torch.from_numpy(np.ascontiguousarray(indptr)).to(dev),
        torch.from_numpy(np.ascontiguousarray(indices)).to(dev),
        torch.from_numpy(np.ascontiguousarray(data)).to(dev),
        int(rows),
        int(cols),
        int(m.nnz),
    )


def matrix_operand(a, name="a"):
    if isinstance(a, (DenseOperand, SparseOperand)):
        return a
    if sp.issparse(a):
        return sparse_operand(a)
    return dense_operand(a, name)

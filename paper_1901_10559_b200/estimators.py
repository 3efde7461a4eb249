"""The reference's error metric on the device.

Drop-in for ``idsketch.estimators`` (reference ``pkg/src/idsketch/estimators.py``):

* ``est_spectral_norm`` (``estimators.py:26-88``): same algorithm, arguments,
  defaults, random-draw order (``default_rng(seed)``: x, y, starts) and
  ``ValueError``s; the iterates live in HBM.
* ``id_residual_operator`` (``estimators.py:91-110``) and ``matrix_operator``
  (``:113-121``) return device operators whose passes over A are this
  package's kernels (``ids_dense_gemv_f64`` in either layout,
  ``ids_csr_spmv_f64`` on the CSR of A and of A^T).  The residual
  x -> A[:, J](P x) - A x is applied as one pass A (E_J P x - x), and its
  adjoint as (E_J P - I)^T (A^T y): one pass over A per application instead
  of the reference's two products.

Operators from these factories accept and return CUDA float64 vectors (numpy
input is copied over); ``est_spectral_norm`` also accepts plain numpy
callables, which it calls with host vectors.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _device
from ._inputs import matrix_operand
from ._native import call, query

ADJOINT_RTOL = 1e-10  # estimators.py:14


@dataclass(frozen=True)
class NormEstimate:
    """Lower estimate of a spectral norm, with the settings that produced it."""

    value: float
    iterations: int
    probes: int


def derive_seed(master, *tags):
    """Deterministic child seed (reference bench.py:116-120)."""
    words = np.random.SeedSequence([int(master)] + [int(t) for t in tags]).generate_state(1)
    return int(words[0])


class DeviceOperator:
    """A linear map on CUDA float64 vectors (marks the device path)."""

    device_operator = True

    def __init__(self, fn, in_dim, out_dim):
        self._fn = fn
        self.in_dim = int(in_dim)
        self.out_dim = int(out_dim)

    def __call__(self, x):
        x = _vec(x)
        if x.numel() != self.in_dim:
            raise ValueError(f"operator expects a vector of length {self.in_dim}, got {x.numel()}")
        return self._fn(x)


def _vec(x):
    t = _device.to_device(x, torch.float64).reshape(-1)
    return t.contiguous()


class _DeviceMatrix:
    """A (dense or sparse) resident on the device with its two passes."""

    def __init__(self, a):
        op = matrix_operand(a)
        self.rows, self.cols = op.shape
        if op.kind == "dense":
            self.dense = op
            self.csr = self.csr_t = None
        else:
            self.dense = None
            if op.kind == "csr":
                self.csr = (op.indptr, op.indices, op.data)
                self.csr_t = _transpose(op.indptr, op.indices, op.data, op.rows, op.cols, op.nnz)
            else:  # CSC of A is the CSR of A^T
                self.csr_t = (op.indptr, op.indices, op.data)
                self.csr = _transpose(op.indptr, op.indices, op.data, op.cols, op.rows, op.nnz)
            self.nnz = op.nnz

    def matvec(self, x, trans=False):
        """A x (trans False) or A^T x on a CUDA vector."""
        n_out = self.cols if trans else self.rows
        y = _device.empty(n_out, torch.float64)
        if self.dense is not None:
            d = self.dense
            nbytes = query("ids_dense_gemv_workspace_bytes", d.rows, d.cols, d.layout, int(trans))
            ws = _device.workspace(nbytes)
            call("ids_dense_gemv_f64", _device.ptr(d.t), d.rows, d.cols, d.ld, d.layout,
                 int(trans), _device.ptr(x), _device.ptr(y), _device.ptr(ws), nbytes,
                 _device.stream_ptr())
        else:
            indptr, indices, data = self.csr_t if trans else self.csr
            rows, cols = (self.cols, self.rows) if trans else (self.rows, self.cols)
            call("ids_csr_spmv_f64", _device.ptr(indptr), int(indptr.dtype == torch.int64),
                 _device.ptr(indices), _device.ptr(data), rows, cols, self.nnz,
                 _device.ptr(x), _device.ptr(y), _device.stream_ptr())
        return y


def _transpose(indptr, indices, data, rows, cols, nnz):
    t_indptr = _device.empty(cols + 1, torch.int64)
    t_indices = _device.empty(max(nnz, 1), torch.int32)
    t_data = _device.empty(max(nnz, 1), torch.float64)
    nbytes = query("ids_csr_transpose_workspace_bytes", rows, cols, nnz)
    ws = _device.workspace(nbytes)
    call("ids_csr_transpose_f64", _device.ptr(indptr), int(indptr.dtype == torch.int64),
         _device.ptr(indices), _device.ptr(data), rows, cols, nnz, _device.ptr(t_indptr),
         _device.ptr(t_indices), _device.ptr(t_data), _device.ptr(ws), nbytes,
         _device.stream_ptr())
    return t_indptr, t_indices, t_data


def _small_dense(p):
    """Row-major CUDA copy of a small dense matrix wrapped as a _DeviceMatrix."""
    return _DeviceMatrix(_device.to_device(np.ascontiguousarray(p, dtype=np.float64)))


def matrix_operator(a):
    """Operator pair for a plain (sparse or dense) matrix (estimators.py:113-121)."""
    m = _DeviceMatrix(a)
    return (DeviceOperator(lambda x: m.matvec(x), m.cols, m.rows),
            DeviceOperator(lambda y: m.matvec(y, trans=True), m.rows, m.cols))


def id_residual_operator(a, decomp):
    """Operator pair for the ID residual x -> A[:, cols] (coeffs @ x) - A x
    (estimators.py:91-110); never forms the residual matrix."""
    m = _DeviceMatrix(a)
    coeffs = np.asarray(decomp.coeffs, dtype=np.float64)
    cols = torch.as_tensor(np.asarray(decomp.cols, dtype=np.int64), device=_device.device())
    if coeffs.ndim != 2 or coeffs.shape[1] != m.cols or coeffs.shape[0] != cols.numel():
        raise ValueError("decomposition does not match the matrix")
    p = _small_dense(coeffs)

    def apply(x):
        u = -x
        u.index_add_(0, cols, p.matvec(x))        # E_J (P x) - x
        return m.matvec(u)

    def apply_adjoint(y):
        z = m.matvec(y, trans=True)               # A^T y
        out = p.matvec(z.index_select(0, cols).contiguous(), trans=True)
        return out.sub_(z)                        # P^T (A^T y)[J] - A^T y

    return DeviceOperator(apply, m.cols, m.rows), DeviceOperator(apply_adjoint, m.rows, m.cols)


def _apply(fn, v):
    if getattr(fn, "device_operator", False):
        return fn(v)
    out = fn(v.cpu().numpy())  # a user-supplied host callable
    return _vec(np.asarray(out, dtype=np.float64))


def _norm(v):
    return float(torch.linalg.vector_norm(v))


def est_spectral_norm(apply, apply_adjoint, cols, iters=10, probes=2, seed=None):
    """Lower estimate of the spectral norm of the operator pair by power
    iteration on the normal operator (estimators.py:26-88)."""
    if cols < 1:
        raise ValueError("cols must be positive")
    if iters < 0 or probes < 1:
        raise ValueError("need iters >= 0 and probes >= 1")
    rng = np.random.default_rng(seed)

    x = _vec(rng.standard_normal(cols))
    bx = _apply(apply, x)
    y = _vec(rng.standard_normal(bx.numel()))
    bty = _apply(apply_adjoint, y)
    lhs = float(torch.dot(bx, y))
    rhs = float(torch.dot(x, bty))
    scale = _norm(bx) * _norm(y) + _norm(x) * _norm(bty)
    if abs(lhs - rhs) > ADJOINT_RTOL * max(scale, 1.0):
        raise ValueError(
            f"operator pair failed the adjoint test: <Bx, y>={lhs!r} vs <x, B'y>={rhs!r}"
        )

    starts = rng.standard_normal((probes, cols))
    best = 0.0
    for p in range(probes):
        v = _vec(starts[p])
        norm_v = _norm(v)
        if norm_v == 0.0:
            continue
        v = v / norm_v
        for _ in range(iters):
            v = _apply(apply_adjoint, _apply(apply, v))
            norm_v = _norm(v)
            if norm_v == 0.0:
                break
            v = v / norm_v
        nv = _norm(v)
        if nv == 0.0:
            continue
        best = max(best, _norm(_apply(apply, v)) / nv)
    return NormEstimate(value=best, iterations=iters, probes=probes)

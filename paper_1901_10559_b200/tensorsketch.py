"""Device TensorSketch launcher (ids_tensorsketch_f64).

Replaces reference sketch.py:156-186: per mode, CountSketch the factor
columns, length-L FFT, spectrum product across modes, inverse FFT, x weights
-- fused into one kernel that never forms a Khatri-Rao column.
"""

import ctypes

import numpy as np
import scipy.sparse as sp
import torch

from . import _device
from ._native import call, query


def factor_to_device(f):
    """Factor (I_n x R) -> col-major CUDA float64 tensor of shape (R, I_n)."""
    if sp.issparse(f):
        m = sp.csc_array(f)
        dense = _device.zeros((m.shape[1], m.shape[0]), torch.float64)
        if m.nnz:
            cols = np.repeat(np.arange(m.shape[1]), np.diff(m.indptr))
            rows = np.asarray(m.indices, dtype=np.int64)
            flat = torch.from_numpy(cols * m.shape[0] + rows).to(dense.device)
            dense.view(-1).index_put_(
                (flat,), torch.from_numpy(np.asarray(m.data, np.float64)).to(dense.device),
                accumulate=True,
            )
        return dense
    if isinstance(f, torch.Tensor):
        t = f.to(torch.float64)
        if t.device.type != "cuda":
            t = t.to(_device.device())
        return t.t().contiguous()
    arr = np.asarray(f, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError("factor must be 2-D")
    t = torch.from_numpy(np.ascontiguousarray(arr.T))
    # page-locked host memory (e.g. a view of a pinned buffer): an async DMA
    # ordered on the current stream; the caller's array outlives the call,
    # which ends with a synchronizing device->host read
    return t.to(_device.device(), non_blocking=t.is_pinned())


SCATTER_MIN_DIM = 4096  # mode length from which the fused kernel uses a scatter plan
USE_SPLIT = True  # the split-spectrum kernel where it applies (tests flip it to compare)


def uses_split_kernel(n_modes, out_dim):
    """Whether (n_modes, L) runs on the split-spectrum cluster kernel
    (ids_tensorsketch_split_f64: L in {4096, 8192, 16384}, <= 8 modes)."""
    return USE_SPLIT and bool(query("ids_tensorsketch_split_ok", n_modes, out_dim))


def tensorsketch_device(op, factors, weights=None, norms=False):
    """Y = TensorSketch(khatri_rao(factors)) diag(weights): CUDA (R, L) tensor.
    norms=True returns (Y, colnorm2): the fused kernel's epilogue also writes
    ||Y[:, r]||^2 (None on the long-sketch route), which the CPQR takes in
    place of its own first pass over Y."""
    if len(factors) != len(op.mode_ops):
        raise ValueError(f"expected {len(op.mode_ops)} factors, got {len(factors)}")
    ncols = factors[0].shape[1]
    for f in factors:
        if f.shape[1] != ncols:
            raise ValueError("factors must share a column count")
    for f, d in zip(factors, op.mode_dims):
        if f.shape[0] != d:
            raise ValueError(f"factor has {f.shape[0]} rows, mode expects {d}")
    w = None
    if weights is not None:
        if isinstance(weights, torch.Tensor):
            w = weights.to(torch.float64).to(_device.device()).contiguous()
        else:
            wn = np.asarray(weights, dtype=np.float64)
            if wn.shape != (ncols,):
                raise ValueError(f"weights must have length {ncols}, got {wn.shape}")
            w = torch.from_numpy(wn).to(_device.device())
        if tuple(w.shape) != (ncols,):
            raise ValueError(f"weights must have length {ncols}, got {tuple(w.shape)}")
    n = len(factors)
    L = op.out_dim
    if not query("ids_tensorsketch_fused_ok", n, L):
        y = _tensorsketch_spectral(op, factors, w, ncols, L)
        return (y, None) if norms else y
    # Sparse (CSC) factors are never densified: their mode's CountSketch is
    # taken straight from the CSC arrays by the ordered CSC kernel (scipy's
    # order, bit for bit), giving an L x R dense "factor" that the fused
    # kernel then reads through the identity hash of length L -- the same
    # values enter the same FFT as on the dense path (reference sketch.py:175,
    # where scipy sketches the CSC factor directly).
    mode_ops, dev_f = [], []
    for m, f in zip(op.mode_ops, factors):
        if sp.issparse(f):
            from ._inputs import sparse_operand

            dev_f.append(m.apply_device(sparse_operand(sp.csc_array(f, dtype=np.float64))))
            mode_ops.append(_identity_op(L))
        else:
            dev_f.append(factor_to_device(f))
            mode_ops.append(m)
    fac_p = (ctypes.c_void_p * n)(*[_device.ptr(t) for t in dev_f])
    dims = (ctypes.c_int64 * n)(*[int(m.in_dim) for m in mode_ops])
    lds = (ctypes.c_int64 * n)(*[int(t.shape[1]) for t in dev_f])
    y = _device.empty((ncols, L), torch.float64)
    nrm = _device.empty(max(ncols, 1), torch.float64)[:ncols] if norms else None
    if ncols == 0:
        return (y, nrm) if norms else y
    if uses_split_kernel(n, L):
        plans = (ctypes.c_void_p * n)(*[_device.ptr(m._ts_split_plan()) for m in mode_ops])
        call(
            "ids_tensorsketch_split_f64", n, ctypes.addressof(fac_p), ctypes.addressof(dims),
            ctypes.addressof(lds), ncols, ctypes.addressof(plans), L, _device.ptr(w),
            _device.ptr(y), _device.ptr(nrm), _device.stream_ptr(),
        )
        return (y, nrm) if norms else y
    idx = [m._bucket_index() for m in mode_ops]
    # scatter plans pay off on long factor columns; short modes (C4: 1000
    # rows) keep the gather path rather than pay the plan's launches per draw
    plans = (ctypes.c_void_p * n)(*[_device.ptr(m._ts_plan()) if m.in_dim >= SCATTER_MIN_DIM
                                    else None for m in mode_ops])
    ord_p = (ctypes.c_void_p * n)(*[_device.ptr(o) for o, _, _ in idx])
    key_p = (ctypes.c_void_p * n)(*[_device.ptr(k) for _, _, k in idx])
    nbytes = query("ids_tensorsketch_workspace_bytes", n, ctypes.addressof(dims), ncols, L)
    ws = _device.workspace(nbytes)
    call(
        "ids_tensorsketch_planned_f64", n, ctypes.addressof(fac_p), ctypes.addressof(dims),
        ctypes.addressof(lds), ncols, ctypes.addressof(ord_p), ctypes.addressof(key_p),
        ctypes.addressof(plans), L,
        _device.ptr(w), _device.ptr(y), _device.ptr(nrm), _device.ptr(ws), nbytes,
        _device.stream_ptr(),
    )
    # dev_f may be freed now: the caching allocator reuses memory in stream order
    return (y, nrm) if norms else y


_IDENTITY_OPS = {}


def _identity_op(L):
    """CountSketch with bucket = row and sign = +1 on L rows (cached per L and
    device, with its bucket index and scatter plan)."""
    key = (int(L), torch.cuda.current_device())
    op = _IDENTITY_OPS.get(key)
    if op is None:
        from .sketch import CountSketchOp

        op = _IDENTITY_OPS[key] = CountSketchOp.from_arrays(np.arange(L), np.ones(L), out_dim=L)
    return op


SPECTRAL_WORK_BYTES = 3 << 29  # spectrum + FFT ping-pong buffers of one batch of terms (1.5 GB)


def _tensorsketch_spectral(op, factors, w, ncols, L):
    """Transforms longer than the fused kernels hold in shared memory, or
    more modes than they take (sketch.py:170-186 step by step): each mode's
    CountSketch S_n A_n with the dense or CSC kernel (bit-exact, scipy's
    order), then ids_ts_spectral_mode_f64 / ids_ts_spectral_finish_f64 -- a
    hand-written batched Stockham FFT through global memory (two modes'
    real rows per complex transform), spectra multiplied left to right, the inverse folded modulo L, weights applied
    last (the reference's own sequence of operations; no library FFT).  The
    terms are processed in batches sized to SPECTRAL_WORK_BYTES."""
    from ._inputs import dense_operand, sparse_operand
    from ._native import IDS_FLAG_ORDERED

    n = len(factors)
    M = int(query("ids_ts_spectral_len", n, L))
    ys = []
    for mode, f in zip(op.mode_ops, factors):
        if sp.issparse(f):  # CSC sketch straight from the sparse arrays
            y = mode.apply_device(sparse_operand(sp.csc_array(f, dtype=np.float64)))
        else:  # (R, I_n) == col-major I_n x R
            y = mode.apply_device(dense_operand(factor_to_device(f).t()), flags=IDS_FLAG_ORDERED)
        ys.append(y.contiguous())  # (R, L) row-major
    out = _device.empty((ncols, L), torch.float64)
    nb_max = max(1, min(ncols, SPECTRAL_WORK_BYTES // (3 * 16 * M)))
    spec = _device.empty(nb_max * M * 2, torch.float64)
    work = _device.empty(nb_max * M * 4, torch.float64)
    for c0 in range(0, ncols, nb_max):
        nb = min(nb_max, ncols - c0)
        for m in range(0, n - 1, 2):  # two modes per complex transform
            call("ids_ts_spectral_pair_f64", _device.ptr(ys[m][c0:c0 + nb]),
                 _device.ptr(ys[m + 1][c0:c0 + nb]), nb, L, M, _device.ptr(spec),
                 _device.ptr(work), int(m == 0), _device.stream_ptr())
        if n % 2:
            call("ids_ts_spectral_mode_f64", _device.ptr(ys[-1][c0:c0 + nb]), nb, L, M,
                 _device.ptr(spec), _device.ptr(work), int(n == 1), _device.stream_ptr())
        call("ids_ts_spectral_finish_f64", _device.ptr(spec), nb, L, M,
             _device.ptr(w[c0:c0 + nb]) if w is not None else None, _device.ptr(work),
             _device.ptr(out[c0:c0 + nb]), _device.stream_ptr())
    return out

"""Matrix Market and CP-directory I/O feeding the path.

Drop-ins for reference ``mmio.py:15-28`` (``read_matrix_market``,
``write_matrix_market``) and ``cp_tensor.py:329-361`` (``save_cp_dir``,
``load_cp_dir``).  Reading goes through the library's multi-threaded native
parser (``ids_mm_info`` / ``ids_mm_read``, csrc/mmio.cpp); symmetric storage
is expanded the way scipy.io.mmread does, and the result is canonicalized
like the reference's ``as_csc`` / ``as_dense`` (linalg.py:22-53): CSC with
sorted indices, duplicates summed, explicit zeros removed, finite values.
``read_matrix_market_device`` returns the canonical matrix already in HBM
(CSR or dense) for the sketch kernels.  Writing is plain host I/O and uses
scipy's writer exactly as the reference does (17 significant digits).
"""

import ctypes
import json
import os
from pathlib import Path

import numpy as np
import scipy.sparse as sp

from ._native import IDS_OK, check, load

_THREADS = max(1, min(32, os.cpu_count() or 1))


def _info(path):
    lib = load()
    rows, cols, entries = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    kind = (ctypes.c_int32 * 3)()
    rc = lib.ids_mm_info(os.fsencode(path), ctypes.addressof(rows), ctypes.addressof(cols),
                         ctypes.addressof(entries), ctypes.addressof(kind))
    if rc != IDS_OK:
        check(rc, "ids_mm_info")
    return rows.value, cols.value, entries.value, tuple(kind)


def _read_raw(path):
    rows, cols, entries, kind = _info(path)
    fmt, field, sym = kind
    if field == 3:
        raise ValueError("complex Matrix Market files are not supported (the path is real fp64)")
    n = max(entries, 1)
    r = np.empty(n if fmt == 0 else 1, dtype=np.int64)
    c = np.empty(n if fmt == 0 else 1, dtype=np.int64)
    v = np.empty(n, dtype=np.float64)
    got = ctypes.c_int64()
    rc = load().ids_mm_read(os.fsencode(path), _THREADS, r.ctypes.data, c.ctypes.data,
                            v.ctypes.data, n, ctypes.addressof(got))
    if rc != IDS_OK:
        check(rc, "ids_mm_read")
    k = got.value
    return rows, cols, fmt, sym, r[:k], c[:k], v[:k]


def _canonical_csc(m):
    """linalg.py:39-53 (as_csc)."""
    out = sp.csc_array(m, dtype=np.float64)
    out.sum_duplicates()
    out.eliminate_zeros()
    out.sort_indices()
    if out.nnz and not np.isfinite(out.data).all():
        raise ValueError("a contains non-finite entries")
    return out


def read_matrix_market(path):
    """Read a matrix: CSC if coordinate, F-ordered ndarray if array (mmio.py:23-28)."""
    rows, cols, fmt, sym, r, c, v = _read_raw(path)
    if fmt == 0:
        if sym != 0:  # expand like scipy.io.mmread: mirrored off-diagonal entries
            off = r != c
            sign = -1.0 if sym == 2 else 1.0
            r, c, v = (np.concatenate([r, c[off]]), np.concatenate([c, r[off]]),
                       np.concatenate([v, sign * v[off]]))
        return _canonical_csc(sp.coo_array((v, (r, c)), shape=(rows, cols)))
    a = np.zeros((rows, cols), order="F")
    if sym == 0:
        a[:] = v.reshape((cols, rows)).T
    else:  # lower triangle stored column by column (diagonal skipped if skew)
        k = 0
        for j in range(cols):
            lo = j + 1 if sym == 2 else j
            a[lo:, j] = v[k:k + rows - lo]
            k += rows - lo
        strict = np.tril(a, -1)
        a += (-strict.T if sym == 2 else strict.T)
    if a.size == 0:
        raise ValueError("a must be nonempty")
    if not np.isfinite(a).all():
        raise ValueError("a contains non-finite entries")
    return a


def read_matrix_market_device(path):
    """read_matrix_market with the canonical result moved to the device:
    a SparseOperand (CSR) for coordinate files, a CUDA tensor for arrays."""
    import torch

    from . import _device
    from ._inputs import SparseOperand

    m = read_matrix_market(path)
    if not sp.issparse(m):
        return _device.to_device(np.ascontiguousarray(m), torch.float64)
    csr = sp.csr_array(m)
    dev = _device.device()
    return SparseOperand(
        "csr",
        torch.from_numpy(csr.indptr.astype(np.int64)).to(dev),
        torch.from_numpy(csr.indices.astype(np.int32)).to(dev),
        torch.from_numpy(csr.data.astype(np.float64)).to(dev),
        int(csr.shape[0]), int(csr.shape[1]), int(csr.nnz),
    )


def write_matrix_market(path, a):
    """Coordinate format if sparse, array if dense, 17 significant digits
    (mmio.py:15-20)."""
    from scipy.io import mmwrite

    from .linalg import as_dense

    if sp.issparse(a):
        mmwrite(path, _canonical_csc(a), precision=17, symmetry="general")
    else:
        mmwrite(path, as_dense(a), precision=17, symmetry="general")


def save_cp_dir(path, x):
    """meta.json, svalues.txt (17 significant digits) and factor_n.mtx
    (cp_tensor.py:329-343)."""
    path = Path(path)
    path.mkdir(parents=True, exist_ok=True)
    meta = {"n_modes": len(x.factors), "rank": x.rank, "mode_dims": list(x.mode_dims)}
    (path / "meta.json").write_text(json.dumps(meta, indent=2) + "\n")
    (path / "svalues.txt").write_text("".join(f"{w:.17g}\n" for w in x.weights))
    for n, f in enumerate(x.factors, start=1):
        write_matrix_market(path / f"factor_{n}.mtx", f)


def load_cp_dir(path):
    """Read a CP directory; factor columns are re-normalized on load
    (cp_tensor.py:346-361)."""
    from .cp_tensor import CpTensor

    path = Path(path)
    meta = json.loads((path / "meta.json").read_text())
    weights = np.array([float(t) for t in (path / "svalues.txt").read_text().split()])
    factors = [read_matrix_market(path / f"factor_{n}.mtx")
               for n in range(1, meta["n_modes"] + 1)]
    x = CpTensor(weights, factors)
    if x.rank != meta["rank"] or list(x.mode_dims) != list(meta["mode_dims"]):
        raise ValueError(f"CP directory {path} is inconsistent with its meta.json")
    return x

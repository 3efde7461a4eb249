"""numpy/scipy restatement of the reference hot path -- TEST INFRASTRUCTURE ONLY.

Every function names the reference lines it restates (paths relative to
``/root/reference/pkg/src/idsketch``).  The third-party kernels are the same
ones the reference reaches: scipy ``csr_matvecs`` / ``csr_matmat`` for S @ A,
pocketfft (``scipy.fft``) for the TensorSketch transforms, LAPACK ``dgeqp3``
(``scipy.linalg.qr(pivoting=True)``) and ``dtrtrs`` (``solve_triangular``) for
the ID.  Hash draws come from the C restatement in ``hash_oracle.c``.

This module is the checker for the CUDA path and the timed CPU baseline of
``bench.py`` (``cpu_baseline``, ``--impl reference``); it is never imported by
the product package.
"""

from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse as sp
from scipy import fft as _fft

from .cs_hash import countsketch_hash, seed_state

RANK_TOL = 1e-12  # linalg.py:15
OVERSAMPLE = 10  # matrix_id.py:20


def _entropy(seed):
    """sketch.py:33-39."""
    if seed is None:
        return np.random.SeedSequence().entropy
    if isinstance(seed, np.random.SeedSequence):
        return seed.entropy
    return int(seed)


def cs_apply(bucket, sign, out_dim, a):
    """S @ A exactly as sketch.py:108-122 evaluates it (scipy CSR product)."""
    n = bucket.size
    s = sp.csr_array(
        (np.asarray(sign, np.float64), (np.asarray(bucket, np.int64), np.arange(n))),
        shape=(out_dim, n),
    )
    out = s @ a
    if sp.issparse(out):
        out = out.toarray()
    return np.asarray(out, dtype=np.float64)


class OracleCountSketch:
    """sketch.py:51-125 with the hash from hash_oracle.c."""

    def __init__(self, in_dim, out_dim, seed=None, surjective=False, mode=None):
        if in_dim < 1 or out_dim < 1:
            raise ValueError("dimensions must be positive")
        if surjective and out_dim > in_dim:
            raise ValueError("surjective mode requires out_dim <= in_dim")
        state, inc = seed_state(seed, mode)
        self.bucket, self.sign, self.draws = countsketch_hash(
            in_dim, out_dim, state, inc, surjective
        )
        self.in_dim, self.out_dim, self.surjective = int(in_dim), int(out_dim), surjective

    def apply(self, a):
        if a.shape[0] != self.in_dim:
            raise ValueError("row mismatch")
        return cs_apply(self.bucket, self.sign, self.out_dim, a)


class OracleTensorSketch:
    """sketch.py:128-186: per-mode standard CountSketches seeded
    SeedSequence([entropy, n]); rfft / product / irfft / weights."""

    def __init__(self, mode_dims, out_dim, seed=None):
        self.mode_dims = tuple(int(d) for d in mode_dims)
        self.out_dim = int(out_dim)
        self.seed = _entropy(seed)
        self.mode_ops = [
            OracleCountSketch(d, out_dim, self.seed, surjective=False, mode=n)
            for n, d in enumerate(self.mode_dims)
        ]

    def apply(self, factors, weights=None):
        return tensorsketch_apply(self.mode_ops, self.out_dim, factors, weights)


def tensorsketch_apply(mode_ops, out_dim, factors, weights=None):
    """sketch.py:156-186."""
    spectrum = None
    for op, f in zip(mode_ops, factors):
        t = _fft.rfft(cs_apply(op.bucket, op.sign, out_dim, f), axis=0)
        spectrum = t if spectrum is None else spectrum * t
    out = _fft.irfft(spectrum, n=out_dim, axis=0)
    if weights is not None:
        out = out * np.asarray(weights, dtype=np.float64)
    return out


@dataclass
class OracleQr:
    q: np.ndarray
    r: np.ndarray
    perm: np.ndarray
    numerical_rank: int


def cpqr(a, rank, rank_tol=RANK_TOL):
    """linalg.py:76-103 (LAPACK dgeqp3 through scipy, then truncation)."""
    a = np.asfortranarray(a, dtype=np.float64)
    q, r, perm = scipy.linalg.qr(a, mode="economic", pivoting=True)
    q = np.ascontiguousarray(q[:, :rank])
    r = np.ascontiguousarray(r[:rank, :])
    d = np.abs(np.diag(r))
    nr = 0 if d[0] == 0.0 else int(np.count_nonzero(d > rank_tol * d[0]))
    return OracleQr(q, r, perm, nr)


def coeffs_from_pivoted(r, perm, rank, numerical_rank, rank_tol=RANK_TOL):
    """matrix_id.py:56-84: floor small diagonals, T = R11^-1 R12, identity scatter."""
    ncols = perm.size
    r11 = np.array(r[:rank, :rank])
    r12 = r[:rank, rank:]
    deficient = numerical_rank < rank
    lead = abs(r11[0, 0])
    if lead == 0.0:
        t = np.zeros((rank, ncols - rank))
    else:
        if deficient:
            floor = rank_tol * lead
            d = np.diag(r11).copy()
            idx = np.flatnonzero(np.abs(d) < floor)
            r11[idx, idx] = np.where(d[idx] < 0.0, -floor, floor)
        if ncols > rank:
            t = scipy.linalg.solve_triangular(r11, r12, lower=False)
        else:
            t = np.zeros((rank, 0))
    coeffs = np.zeros((rank, ncols))
    coeffs[np.arange(rank), perm[:rank]] = 1.0
    coeffs[:, perm[rank:]] = t
    return coeffs, deficient


@dataclass
class OracleId:
    cols: np.ndarray
    coeffs: np.ndarray
    numerical_rank: int
    rank_deficient: bool
    sketch: np.ndarray = None


def matrix_id(y, rank, rank_tol=RANK_TOL):
    """matrix_id.py:87-113."""
    f = cpqr(y, rank, rank_tol)
    coeffs, deficient = coeffs_from_pivoted(f.r, f.perm, rank, f.numerical_rank, rank_tol)
    return OracleId(f.perm[:rank].copy(), coeffs, f.numerical_rank, deficient)


def as_dense(a, name="a"):
    """linalg.py:22-36: F-ordered float64 copy + shape / finiteness checks."""
    out = np.asfortranarray(a, dtype=np.float64)
    if out.ndim != 2 or out.size == 0:
        raise ValueError(f"{name} must be a nonempty 2-D array")
    if not np.isfinite(out).all():
        raise ValueError(f"{name} contains non-finite entries")
    return out


def countsketch_id(a, rank, sketch_dim=None, seed=None, rank_tol=RANK_TOL, surjective=True):
    """matrix_id.py:162-182 (validation of check_matrix_id_args :116-141);
    dense input goes through as_dense like the reference (matrix_id.py:163)."""
    if not sp.issparse(a):
        a = as_dense(a)
    rows, ncols = a.shape
    if not 1 <= rank <= ncols:
        raise ValueError("rank out of range")
    if sketch_dim is None:
        sketch_dim = rank + OVERSAMPLE
    if sketch_dim < rank or sketch_dim >= rows:
        raise ValueError("sketch dimension out of range")
    op = OracleCountSketch(rows, sketch_dim, seed, surjective=surjective)
    y = op.apply(a)
    out = matrix_id(y, rank, rank_tol)
    out.sketch = y
    return out


def ts_new_weights(weights, cols, coeffs):
    """cp_tensor.py:216."""
    return weights[cols] * coeffs.sum(axis=1)


def tensorsketch_id(weights, factors, rank, sketch_dim=None, seed=None, rank_tol=RANK_TOL):
    """cp_tensor.py:242-276 on already-normalized (weights, factors)."""
    dims = [f.shape[0] for f in factors]
    if sketch_dim is None:
        sketch_dim = rank + OVERSAMPLE
    op = OracleTensorSketch(dims, sketch_dim, seed)
    y = op.apply(factors, weights)
    out = matrix_id(y, rank, rank_tol)
    out.sketch = y
    return out, ts_new_weights(np.asarray(weights), out.cols, out.coeffs)


def _dense(f):
    return f.toarray() if sp.issparse(f) else np.asarray(f)


def cp_gram(weights, factors):
    """cp_tensor.py:144-160: diag(w) (hadamard of factor Grams) diag(w)."""
    w = np.asarray(weights, dtype=np.float64)
    out = np.ones((w.size, w.size))
    for f in factors:
        f = _dense(f)
        out *= f.T @ f
    return out * w[None, :] * w[:, None]


def cp_norm(weights, factors):
    """cp_tensor.py:169-172."""
    return float(np.sqrt(max(cp_gram(weights, factors).sum(), 0.0)))


def cp_diff_norm(w1, f1, w2, f2):
    """cp_tensor.py:183-197: || X - Y ||_F through the Gram identity."""
    w = np.concatenate([np.asarray(w1, float), -np.asarray(w2, float)])
    fs = [np.hstack([_dense(a), _dense(b)]) for a, b in zip(f1, f2)]
    return float(np.sqrt(max(cp_gram(w, fs).sum(), 0.0)))

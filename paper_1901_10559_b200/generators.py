"""Seeded synthetic inputs of the BASELINE.json configs, built on the device.

The reference's own generators (``pkg/src/idsketch/generators.py:12-107``:
sparse rank-1 sums with a spectral knee) are not what BASELINE.json quotes its
configs on; these functions restate the five configs of BASELINE.json as
SURVEY.md section 8(d) reads them, on the GPU and shardable:

* ``dense_config("C1" | "C2")``: A = U diag(sigma) V^T (+ iid noise), U the
  orthonormal factor of a seeded N(0, 1) rows x cols matrix, V that of a
  seeded cols x cols one.  U is orthonormalized by Cholesky QR over fixed
  global row chunks (G = U R, R from chol(G^T G)), so any contiguous row block
  of A can be built on its own rank and every world size builds the same
  global matrix.  C2's noise is read as variance 1e-8 (std 1e-4).
* ``csr_config("C3")``: CSR rows x cols with uniformly random positions
  (row lengths Poisson(nnz_per_row), distinct sorted columns per row) and
  the planted structure of SURVEY.md 8(d): a latent Z (rows x 20) ~ N(0, 1);
  column j < 20 holds Z[:, j] on its pattern, column c >= 20 holds
  (Z w_c) on its pattern with w_c ~ N(0, I_20).  int32 indptr / indices,
  as scipy picks for 1e8 nonzeros.
* ``cp_config("C4" | "C5")``: near-duplicate CP terms -- terms 0..B-1 have
  unit-norm N(0, 1) factor columns, term r >= B copies a seeded base
  c_r in [0, B): a_r = normalize(a_{c_r} + pert * g); weights ~ U(0.5, 1).

Every generator takes a ``seed`` (default: the config number) and a row or
term range; blocks of the same seed agree bit for bit with the whole.
These feed ``bench.py`` and the config-shape parity tests; they are input
plumbing, not part of the sketch path.
"""

import numpy as np
import torch

from . import _device
from ._inputs import SparseOperand

CONFIGS = {
    # dense: rows, cols, low rank, tail law, noise std, K, L
    "C1": dict(kind="dense", rows=10_000, cols=1_000, lowrank=10, tail="pow10", noise=0.0,
               k=10, L=40),
    "C2": dict(kind="dense", rows=1_000_000, cols=2_000, lowrank=20, tail="geom0.9",
               noise=1e-4, k=20, L=100),
    # sparse: rows, cols, mean nonzeros per row, latent rank, K, L
    "C3": dict(kind="csr", rows=10_000_000, cols=10_000, per_row=10, latent=20, k=20, L=200),
    # CP: modes, mode length, terms, base terms, perturbation, K, L
    "C4": dict(kind="cp", modes=3, dim=1_000, terms=1_000, bases=10, pert=1e-3, k=10, L=4096),
    "C5": dict(kind="cp", modes=4, dim=10_000, terms=2_000, bases=20, pert=1e-4, k=20,
               L=16384),
}

DENSE_CHUNK = 125_000  # global rows per generator chunk (C2: 8 chunks)
CSR_CHUNK = 250_000  # global rows per generator chunk (C3: 40 chunks)


def default_seed(name):
    return int(name[1:])


def config_sigma(name, cols=None):
    """Singular values of the dense configs (BASELINE.json configs[0..1])."""
    c = CONFIGS[name]
    cols = cols or c["cols"]
    i = np.arange(1, cols + 1, dtype=np.float64)
    k = c["lowrank"]
    if c["tail"] == "pow10":
        tail = 10.0 ** (-(i - k) / 10.0)
    else:
        tail = 0.9 ** (i - k)
    return np.where(i <= k, 1.0, tail)


def _gen(dev, *tags):
    g = torch.Generator(device=dev)
    words = np.random.SeedSequence([int(t) for t in tags]).generate_state(2, np.uint32)
    g.manual_seed(int(words[0]) | (int(words[1]) << 32))
    return g


def dense_config(name="C2", rows=None, cols=None, row_range=None, seed=None, layout="C",
                 device=None):
    """Rows [r0, r1) of the dense config matrix as a CUDA float64 tensor
    (C order by default, ``layout="F"`` for column-major)."""
    c = CONFIGS[name]
    if c["kind"] != "dense":
        raise ValueError(f"{name} is not a dense config")
    rows = int(rows or c["rows"])
    cols = int(cols or c["cols"])
    seed = default_seed(name) if seed is None else int(seed)
    r0, r1 = row_range or (0, rows)
    dev = torch.device(device) if device is not None else _device.device()
    # V: orthonormal factor of a seeded cols x cols Gaussian
    gv = _gen(dev, seed, 1)
    v = torch.linalg.qr(torch.randn(cols, cols, generator=gv, device=dev,
                                    dtype=torch.float64))[0]
    sig = torch.from_numpy(config_sigma(name, cols)).to(dev)
    nchunks = -(-rows // DENSE_CHUNK)

    def chunk(ci):
        n = min(DENSE_CHUNK, rows - ci * DENSE_CHUNK)
        g = _gen(dev, seed, 2, ci)
        return g, torch.randn(n, cols, generator=g, device=dev, dtype=torch.float64)

    # Cholesky QR: G = U Rc with U orthonormal; the Gram needs every chunk
    gram = torch.zeros(cols, cols, dtype=torch.float64, device=dev)
    for ci in range(nchunks):
        _, gch = chunk(ci)
        gram.addmm_(gch.t(), gch)
        del gch
    rc = torch.linalg.cholesky(gram, upper=True)
    # A rows = G Rc^-1 diag(sigma) V^T
    m = torch.linalg.solve_triangular(rc, torch.diag(sig) @ v.t(), upper=True)
    if layout == "F":
        out = torch.empty((cols, r1 - r0), dtype=torch.float64, device=dev).t()
    else:
        out = torch.empty((r1 - r0, cols), dtype=torch.float64, device=dev)
    for ci in range(r0 // DENSE_CHUNK, -(-r1 // DENSE_CHUNK)):
        c0 = ci * DENSE_CHUNK
        g, gch = chunk(ci)
        blk = gch @ m
        if c["noise"] > 0:
            blk.add_(torch.randn(blk.shape, generator=g, device=dev, dtype=torch.float64),
                     alpha=c["noise"])
        a, b = max(c0, r0), min(c0 + gch.shape[0], r1)
        out[a - r0:b - r0] = blk[a - c0:b - c0]
        del gch, blk
    return out


def _csr_chunk(dev, seed, ci, n, cols, per_row, wt):
    """One generator chunk of the C3 matrix: (row lengths, columns, values)."""
    g = _gen(dev, seed, 3, ci)
    counts = torch.poisson(torch.full((n,), float(per_row), device=dev, dtype=torch.float64),
                           generator=g).to(torch.int64).clamp_(max=cols)
    nnz = int(counts.sum())
    row = torch.repeat_interleave(torch.arange(n, device=dev), counts)
    col = torch.randint(0, cols, (nnz,), generator=g, device=dev)
    key = torch.sort(row * cols + col).values
    while True:  # distinct columns within a row: redraw duplicates
        dup = torch.nonzero(key[1:] == key[:-1]).flatten() + 1
        if dup.numel() == 0:
            break
        r = key[dup] // cols
        key[dup] = r * cols + torch.randint(0, cols, (dup.numel(),), generator=g, device=dev)
        key = torch.sort(key).values
    row, col = key // cols, key % cols
    z = torch.randn(n, wt.shape[1], generator=g, device=dev, dtype=torch.float64)
    vals = torch.empty(nnz, dtype=torch.float64, device=dev)
    step = 1 << 22
    for s in range(0, nnz, step):
        e = min(nnz, s + step)
        vals[s:e] = (z[row[s:e]] * wt[col[s:e]]).sum(1)
    return counts, col.to(torch.int32), vals


def csr_config(name="C3", rows=None, cols=None, row_range=None, seed=None, device=None):
    """Rows [r0, r1) of the C3 CSR matrix as a device ``SparseOperand``
    (local row numbering, int32 indptr / indices, float64 data)."""
    c = CONFIGS[name]
    if c["kind"] != "csr":
        raise ValueError(f"{name} is not a sparse config")
    rows = int(rows or c["rows"])
    cols = int(cols or c["cols"])
    seed = default_seed(name) if seed is None else int(seed)
    r0, r1 = row_range or (0, rows)
    dev = torch.device(device) if device is not None else _device.device()
    lat = min(c["latent"], cols)
    # column weights: w_c = e_c for c < latent, N(0, I) beyond
    gw = _gen(dev, seed, 4)
    wt = torch.randn(cols, lat, generator=gw, device=dev, dtype=torch.float64)
    wt[:lat] = torch.eye(lat, dtype=torch.float64, device=dev)
    counts, idx, val = [], [], []
    for ci in range(r0 // CSR_CHUNK, -(-r1 // CSR_CHUNK)):
        c0 = ci * CSR_CHUNK
        n = min(CSR_CHUNK, rows - c0)
        cnt, col, v = _csr_chunk(dev, seed, ci, n, cols, c["per_row"], wt)
        a, b = max(c0, r0) - c0, min(c0 + n, r1) - c0
        ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
        torch.cumsum(cnt, 0, out=ptr[1:])
        s, e = int(ptr[a]), int(ptr[b])
        counts.append(cnt[a:b])
        idx.append(col[s:e])
        val.append(v[s:e])
    counts = torch.cat(counts)
    nnz = int(counts.sum())
    ptr_dtype = torch.int32 if nnz < 2**31 else torch.int64
    indptr = torch.zeros(r1 - r0 + 1, dtype=ptr_dtype, device=dev)
    indptr[1:] = torch.cumsum(counts, 0).to(ptr_dtype)
    return SparseOperand("csr", indptr, torch.cat(idx), torch.cat(val), r1 - r0, cols, nnz,
                         host=False)


def cp_config(name="C5", col_range=None, seed=None, dim=None, terms=None, device=None):
    """Terms [c0, c1) of the C4 / C5 CP tensor: (weights CUDA (R_local,),
    factors: list of CUDA I_n x R_local column-major views)."""
    c = CONFIGS[name]
    if c["kind"] != "cp":
        raise ValueError(f"{name} is not a CP config")
    dim = int(dim or c["dim"])
    R = int(terms or c["terms"])
    nb = min(c["bases"], R)
    seed = default_seed(name) if seed is None else int(seed)
    c0, c1 = col_range or (0, R)
    dev = torch.device(device) if device is not None else _device.device()
    g = _gen(dev, seed, 5)
    base = torch.randint(0, nb, (R,), generator=g, device=dev)
    base[:nb] = torch.arange(nb, device=dev)
    facs = []
    for _ in range(c["modes"]):
        b = torch.randn(nb, dim, generator=g, device=dev, dtype=torch.float64)
        b /= torch.linalg.vector_norm(b, dim=1, keepdim=True)
        f = b[base] + c["pert"] * torch.randn(R, dim, generator=g, device=dev,
                                              dtype=torch.float64)  # row r = term r
        f /= torch.linalg.vector_norm(f, dim=1, keepdim=True)
        f[:nb] = b  # the base terms themselves are unperturbed
        facs.append(f[c0:c1].contiguous().t())  # I_n x R_local, column-major
    w = torch.rand(R, generator=g, device=dev, dtype=torch.float64) * 0.5 + 0.5
    return w[c0:c1].contiguous(), facs


def operand_to_scipy(op):
    """Device CSR/CSC SparseOperand -> scipy sparse array on the host."""
    import scipy.sparse as sp

    cls = sp.csr_array if op.fmt == "csr" else sp.csc_array
    return cls((op.data.cpu().numpy(), op.indices.cpu().numpy(), op.indptr.cpu().numpy()),
               shape=(op.rows, op.cols))


__all__ = ["CONFIGS", "config_sigma", "cp_config", "csr_config", "default_seed",
           "dense_config", "operand_to_scipy"]

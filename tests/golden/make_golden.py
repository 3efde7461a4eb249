"""Generate the golden fixtures from the REAL reference package.

Run here (the container that has /root/reference):

    python tests/golden/make_golden.py

It imports ``idsketch`` from /root/reference/pkg/src (read-only, never copied)
and writes ``tests/golden/golden.npz`` plus ``tests/golden/manifest.json``.
The fixtures pin the oracle (tests/test_oracle_golden.py) and the CUDA path
(tests/test_gpu_parity.py).  Large hash draws are pinned by SHA-256 digests of
the int64 bucket / float64 sign bytes so they stay small.

Pinned toolchain: numpy 2.3.5, scipy 1.18.1 (Python 3.12.3).
"""

import hashlib
import json
import os
import sys

import numpy as np
import scipy
import scipy.sparse as sp

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from idsketch.bench import derive_seed  # noqa: E402
from idsketch.cp_tensor import CpTensor, cp_diff_norm, cp_norm, tensorsketch_id  # noqa: E402
from idsketch.estimators import (  # noqa: E402
    est_spectral_norm, id_residual_operator, matrix_operator)
from idsketch.matrix_id import countsketch_id, matrix_id, matrix_sketch  # noqa: E402
from idsketch.sketch import CountSketchOp, TensorSketchOp  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def spectrum_matrix(rng, rows, cols, sigma):
    u = np.linalg.qr(rng.standard_normal((rows, len(sigma))))[0]
    v = np.linalg.qr(rng.standard_normal((cols, len(sigma))))[0]
    return (u * sigma) @ v.T


def main():
    arrays = {}
    manifest = {
        "numpy": np.__version__,
        "scipy": scipy.__version__,
        "hash_small": [],
        "hash_digest": [],
        "sketch_dense": [],
        "sketch_csr": [],
        "tensorsketch": [],
        "matrix_id": [],
        "countsketch_id": [],
        "tensorsketch_id": [],
        "error_estimates": [],
    }

    # ---- hash: full arrays for small cases -------------------------------
    small = [
        (4, 4, 0, True), (1000, 10, 1, True), (10000, 40, 3, True),
        (73, 9, 5, False), (30, 7, 99, True), (100, 1, 3, False),
        (100, 1, 3, True), (5, 5, 2, True), (1, 1, 0, False), (1, 1, 0, True),
        (2, 1, 4, True), (3000, 2999, 6, True), (4097, 64, 12, True),
        (777, 5, 13, False), (20011, 1000, 14, True),
    ]
    for n, (I, L, seed, surj) in enumerate(small):
        op = CountSketchOp(I, L, seed=seed, surjective=surj)
        arrays[f"hash{n}_bucket"] = op.bucket.astype(np.int64)
        arrays[f"hash{n}_sign"] = op.sign.astype(np.float64)
        manifest["hash_small"].append(
            {"id": n, "in_dim": I, "out_dim": L, "seed": seed, "surjective": surj}
        )

    # ---- hash: digests for the BASELINE.json config sizes -----------------
    big = [(10_000, 40, s, True) for s in range(10)]
    big += [(1_000_000, 100, s, True) for s in range(3)]
    big += [(10_000_000, 200, 0, True)]
    big += [(1_000_000, 100, 5, False), (2**21 + 17, 333, 8, True)]
    for I, L, seed, surj in big:
        op = CountSketchOp(I, L, seed=seed, surjective=surj)
        manifest["hash_digest"].append(
            {"in_dim": I, "out_dim": L, "seed": seed, "surjective": surj,
             "mode": None, "sha256": digest(op.bucket.astype(np.int64),
                                            op.sign.astype(np.float64))}
        )
    for dims, L, seed in (([1000] * 3, 4096, 0), ([10_000] * 4, 16384, 0),
                          ([1000] * 3, 4096, 7)):
        ts = TensorSketchOp(dims, L, seed=seed)
        for mode, op in enumerate(ts.mode_ops):
            manifest["hash_digest"].append(
                {"in_dim": dims[mode], "out_dim": L, "seed": seed, "surjective": False,
                 "mode": mode, "sha256": digest(op.bucket.astype(np.int64),
                                                op.sign.astype(np.float64))}
            )

    # ---- CountSketch apply: dense (both orders) and CSR --------------------
    rng = np.random.default_rng(2024)
    for n, (I, R, L, seed, surj) in enumerate(
        [(200, 30, 17, 0, True), (1000, 64, 40, 1, False), (57, 3, 56, 2, True),
         (1500, 65, 100, 3, True)]
    ):
        a = rng.standard_normal((I, R))
        op = CountSketchOp(I, L, seed=seed, surjective=surj)
        arrays[f"sd{n}_a"] = a
        arrays[f"sd{n}_y"] = op.apply(a)
        manifest["sketch_dense"].append(
            {"id": n, "in_dim": I, "cols": R, "out_dim": L, "seed": seed, "surjective": surj}
        )
    for n, (I, R, L, dens, seed, surj) in enumerate(
        [(500, 40, 30, 0.05, 4, True), (2000, 300, 64, 0.01, 5, False),
         (100, 15, 20, 0.05, 4, False)]
    ):
        a = sp.random_array((I, R), density=dens, rng=rng, format="csr")
        op = CountSketchOp(I, L, seed=seed, surjective=surj)
        arrays[f"sc{n}_indptr"] = a.indptr.astype(np.int64)
        arrays[f"sc{n}_indices"] = a.indices.astype(np.int32)
        arrays[f"sc{n}_data"] = a.data
        arrays[f"sc{n}_y"] = op.apply(a)
        manifest["sketch_csr"].append(
            {"id": n, "in_dim": I, "cols": R, "out_dim": L, "seed": seed, "surjective": surj}
        )

    # ---- TensorSketch apply ------------------------------------------------
    for n, (dims, R, L, seed) in enumerate(
        [([12], 5, 8, 8), ([3, 3], 2, 4, 1), ([2, 2, 2], 1, 5, 9), ([9, 7, 11], 6, 13, 3),
         ([40, 30, 20], 16, 64, 4), ([100, 90, 80, 70], 12, 256, 5),
         ([300, 200, 100], 20, 1024, 6), ([6, 5], 4, 7, 7)]
    ):
        factors = [rng.standard_normal((d, R)) for d in dims]
        lam = rng.random(R) + 0.5
        ts = TensorSketchOp(dims, L, seed=seed)
        for m, f in enumerate(factors):
            arrays[f"ts{n}_f{m}"] = f
        arrays[f"ts{n}_w"] = lam
        arrays[f"ts{n}_y"] = ts.apply(factors, lam)
        manifest["tensorsketch"].append(
            {"id": n, "dims": dims, "cols": R, "out_dim": L, "seed": seed}
        )

    # ---- matrix_id on small sketches --------------------------------------
    mids = []
    mids.append((np.array([[1.0, 0.0, 2.0], [0.0, 1.0, 3.0]]), 2))
    mids.append((rng.standard_normal((20, 4)) @ rng.standard_normal((4, 15)), 10))
    mids.append((np.zeros((5, 4)), 2))
    mids.append((spectrum_matrix(rng, 40, 25, 2.0 ** -np.arange(25.0)), 10))
    mids.append((rng.standard_normal((40, 300)), 10))
    mids.append((rng.standard_normal((60, 500)), 20))
    mids.append((rng.standard_normal((9, 6)), 6))
    mids.append((rng.standard_normal((6, 9)), 6))
    for n, (y, k) in enumerate(mids):
        d = matrix_id(y, k)
        arrays[f"mid{n}_y"] = y
        arrays[f"mid{n}_cols"] = d.cols
        arrays[f"mid{n}_coeffs"] = d.coeffs
        manifest["matrix_id"].append(
            {"id": n, "rank": k, "numerical_rank": int(d.numerical_rank),
             "rank_deficient": bool(d.rank_deficient)}
        )

    # ---- countsketch_id end to end (C1-shaped but small enough to store) ---
    a_c1 = spectrum_matrix(
        np.random.default_rng(1), 1000, 120,
        np.concatenate([np.ones(10), 10.0 ** (-np.arange(1, 111) / 10.0)]),
    )
    arrays["csid_a"] = a_c1
    for seed in range(10):
        d = countsketch_id(a_c1, 10, 40, seed=seed)
        y = matrix_sketch(a_c1, "countsketch", 40, seed=seed, surjective=True)
        arrays[f"csid{seed}_cols"] = d.cols
        arrays[f"csid{seed}_coeffs"] = d.coeffs
        arrays[f"csid{seed}_y"] = y
        manifest["countsketch_id"].append(
            {"seed": seed, "rank": 10, "sketch_dim": 40,
             "numerical_rank": int(d.numerical_rank)}
        )
        # the reference's own error metric for a matrix trial (bench.py:137-145)
        ap, adj = id_residual_operator(a_c1, d)
        est = est_spectral_norm(ap, adj, cols=a_c1.shape[1], iters=10, probes=2,
                                seed=derive_seed(seed, 0xE57))
        manifest["error_estimates"].append(
            {"case": "csid", "seed": seed, "est_seed": derive_seed(seed, 0xE57),
             "value": est.value})
    a_sp = sp.random_array((3000, 120), density=0.02, rng=np.random.default_rng(3),
                           format="csr")
    arrays["csid_sp_indptr"] = a_sp.indptr.astype(np.int64)
    arrays["csid_sp_indices"] = a_sp.indices.astype(np.int32)
    arrays["csid_sp_data"] = a_sp.data
    d = countsketch_id(a_sp, 12, 50, seed=21)
    arrays["csid_sp_cols"] = d.cols
    arrays["csid_sp_coeffs"] = d.coeffs
    ap, adj = id_residual_operator(a_sp, d)
    est = est_spectral_norm(ap, adj, cols=a_sp.shape[1], seed=derive_seed(21, 0xE57))
    manifest["error_estimates"].append(
        {"case": "csid_sp", "seed": 21, "est_seed": derive_seed(21, 0xE57), "value": est.value})
    ap, adj = matrix_operator(a_c1)
    est = est_spectral_norm(ap, adj, cols=a_c1.shape[1], iters=5, probes=3, seed=7)
    manifest["error_estimates"].append(
        {"case": "matrix_operator", "iters": 5, "probes": 3, "est_seed": 7, "value": est.value})

    # ---- tensorsketch_id (C4-shaped construction, reduced size) ------------
    trng = np.random.default_rng(4)
    dims, R, base, k, L = (60, 50, 40), 120, 6, 6, 512
    fac = []
    bases = trng.integers(0, base, size=R)
    bases[:base] = np.arange(base)
    for d_ in dims:
        f = trng.standard_normal((d_, R))
        f[:, :base] /= np.linalg.norm(f[:, :base], axis=0)
        for r in range(base, R):
            g = f[:, bases[r]] + 1e-3 * trng.standard_normal(d_)
            f[:, r] = g / np.linalg.norm(g)
        fac.append(f)
    w = trng.uniform(0.5, 1.0, size=R)
    x = CpTensor(w, fac)
    res = tensorsketch_id(x, k, L, seed=11)
    for m, f in enumerate(x.factors):
        arrays[f"tsid_f{m}"] = f
    arrays["tsid_w"] = x.weights
    arrays["tsid_cols"] = res.cols
    arrays["tsid_coeffs"] = res.coeffs
    arrays["tsid_new_weights"] = res.new_weights
    manifest["tensorsketch_id"].append(
        {"dims": list(dims), "terms": R, "rank": k, "sketch_dim": L, "seed": 11,
         "numerical_rank": int(res.numerical_rank),
         "cp_diff_norm": cp_diff_norm(x, res.reduced), "cp_norm": cp_norm(x)}
    )

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()

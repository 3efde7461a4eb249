"""Parity at the REAL shapes of BASELINE.json configs[1], [2] and [4] (C2, C3,
C5), on the seeded inputs of ``paper_1901_10559_b200.generators`` -- the
same inputs bench.py times.  Each case runs the product path (device input,
C-ABI kernels) and the pinned CPU oracle (scipy S @ A, pocketfft, LAPACK
dgeqp3 / dtrtrs: the third-party kernels the reference itself calls,
matrix_id.py:170-182, cp_tensor.py:266-276) on the same input and seed, and
checks north_star's bar:

* hash bucket / sign bit-exact;
* Y within 1e-10 relative Frobenius (bit-exact where the kernel keeps
  scipy's summation order: dense input);
* j identical, P within 1e-10 relative Frobenius (new_weights too for CP);
* ID error within 1% of the reference's, with the reference's own metric
  (est_spectral_norm of the ID residual with seed derive_seed(seed, 0xE57),
  reference bench.py:137-145; cp_diff_norm for tensors, bench.py:171).

Each case costs 10-40 s of host time (the oracle at full size) on the GPU box."""

import numpy as np
import pytest

import oracle

from conftest import relerr_fro

pytestmark = pytest.mark.gpu

ids = pytest.importorskip("paper_1901_10559_b200")
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1901_10559_b200 import generators as G  # noqa: E402

TOL = 1e-10


def _matrix_error(a, d, seed):
    """Reference metric (bench.py:137-145) evaluated on the device."""
    apply, adj = ids.id_residual_operator(a, d)
    return ids.est_spectral_norm(apply, adj, a.shape[1], iters=10, probes=2,
                                 seed=ids.derive_seed(seed, 0xE57)).value


def _check_matrix(a_dev, a_host, k, L, seed, y_bit_exact):
    rows, cols = a_host.shape
    op = ids.CountSketchOp(rows, L, seed=seed, surjective=True)
    ref_op = oracle.OracleCountSketch(rows, L, seed, True)
    assert np.array_equal(op.bucket, ref_op.bucket)
    assert np.array_equal(op.sign, ref_op.sign)
    y_ref = oracle.cs_apply(ref_op.bucket, ref_op.sign, L, a_host)
    y = op.apply(a_dev)
    y = y.cpu().numpy() if isinstance(y, torch.Tensor) else y
    if y_bit_exact:
        assert np.array_equal(y, y_ref)
    assert relerr_fro(y, y_ref) <= TOL
    want = oracle.matrix_id(y_ref, k)
    d = ids.countsketch_id(a_dev, k, L, seed=seed)
    assert d.cols.dtype == np.int32 and d.coeffs.shape == (k, cols)
    assert np.array_equal(d.cols, want.cols), (d.cols, want.cols)
    assert relerr_fro(d.coeffs, want.coeffs) <= TOL
    assert d.numerical_rank == want.numerical_rank
    assert d.rank_deficient == want.rank_deficient
    err = _matrix_error(a_dev, d, seed)
    ref = _matrix_error(a_dev, want, seed)
    assert abs(err - ref) <= 0.01 * ref, (err, ref)
    return y


@pytest.fixture(scope="module")
def c2():
    a = G.dense_config("C2")
    yield a
    del a
    torch.cuda.empty_cache()


def test_config2_full_size_vs_oracle(c2):
    """C2: dense 1,000,000 x 2,000, K = 20, L = 100, surjective; C order (the
    bench's layout) and the same matrix in F order (the reference's
    as_dense layout, linalg.py:29) both bit-exact against scipy."""
    cfg = G.CONFIGS["C2"]
    host = c2.cpu().numpy()
    for seed in (0, 1):
        y = _check_matrix(c2, host, cfg["k"], cfg["L"], seed, y_bit_exact=True)
    f = c2.t().contiguous().t()  # same values, column-major
    op = ids.CountSketchOp(cfg["rows"], cfg["L"], seed=1, surjective=True)
    assert np.array_equal(op.apply(f).cpu().numpy(), y)
    d = ids.countsketch_id(f, cfg["k"], cfg["L"], seed=1)
    assert np.array_equal(d.cols, ids.countsketch_id(c2, cfg["k"], cfg["L"], seed=1).cols)


def test_config2_generator_spectrum(c2):
    """The generated C2 has orthonormal U (Cholesky QR): the leading 20
    singular values are 1 up to the noise floor, the tail decays by 0.9."""
    s = torch.linalg.eigvalsh(c2.T @ c2).flip(0).clamp(min=0).sqrt().cpu().numpy()
    assert np.all(np.abs(s[:20] - 1.0) < 0.02)
    assert 0.85 < s[21] / s[20] < 0.95


def test_config3_full_size_vs_oracle():
    """C3: CSR 10,000,000 x 10,000 with ~1e8 nonzeros at uniform random
    positions and the latent rank-20 planted structure, K = 20, L = 200."""
    cfg = G.CONFIGS["C3"]
    a = G.csr_config("C3")
    assert 0.99e8 < a.nnz < 1.01e8 and a.indptr.dtype == torch.int32
    host = G.operand_to_scipy(a)
    for seed in (0,):
        _check_matrix(a, host, cfg["k"], cfg["L"], seed, y_bit_exact=False)
    del a, host
    torch.cuda.empty_cache()


def test_config3_row_blocks_match_whole():
    """Row blocks of C3 (what each rank builds) are slices of the whole."""
    whole = G.operand_to_scipy(G.csr_config("C3", rows=1_000_000))
    part = G.operand_to_scipy(G.csr_config("C3", rows=1_000_000, row_range=(300_000, 700_000)))
    assert (whole[300_000:700_000] != part).nnz == 0


def test_config5_full_size_vs_oracle():
    """C5: 4-way CP, I_n = 10,000, R = 2,000 near-duplicate terms, K = 20,
    L = 16,384 (the tall 16384 x 2000 CPQR included)."""
    cfg = G.CONFIGS["C5"]
    w, facs = G.cp_config("C5")
    x = ids.CpTensor(w.cpu().numpy(), [f.cpu().numpy() for f in facs])
    assert all(f.flags.f_contiguous for f in x.factors)
    seed = 0
    want, nw = oracle.tensorsketch_id(x.weights, x.factors, cfg["k"], cfg["L"], seed=seed)
    y = ids.TensorSketchOp(x.mode_dims, cfg["L"], seed=seed).apply(x.factors, x.weights)
    assert relerr_fro(y, want.sketch) <= TOL
    res = ids.tensorsketch_id(x, cfg["k"], cfg["L"], seed=seed)
    assert np.array_equal(res.cols, want.cols), (res.cols, want.cols)
    assert relerr_fro(res.coeffs, want.coeffs) <= TOL
    assert relerr_fro(res.new_weights, nw) <= TOL
    err = ids.cp_diff_norm(x, res.reduced)
    ref = ids.cp_diff_norm(x, x.select(want.cols, nw))
    assert abs(err - ref) <= 0.01 * ref + 1e-12, (err, ref)


def test_config5_tall_cpqr_vs_lapack():
    """The 16384 x 2000 truncated CPQR alone (cpqr_kernel, the tall path)
    against dgeqp3: same pivots, R rows within 1e-10."""
    rng = np.random.default_rng(55)
    base = rng.standard_normal((16384, 20))
    y = base[:, rng.integers(0, 20, 2000)] + 1e-4 * rng.standard_normal((16384, 2000))
    want = oracle.cpqr(y, 20)
    got = ids.cpqr(y, 20)
    assert np.array_equal(got.perm[:20], want.perm[:20])
    assert relerr_fro(np.abs(got.r[:, :20]), np.abs(want.r[:, :20])) <= TOL

"""Behaviours the reference's own test-suite checks (pkg/tests/test_sketch.py,
test_cp_tensor.py, test_estimators.py), restated with fresh inputs against the
B200 implementation."""

import numpy as np
import pytest
import scipy.sparse as sp
from scipy import stats

import oracle

from conftest import khatri_rao, relerr_fro

pytestmark = pytest.mark.gpu

ids = pytest.importorskip("paper_1901_10559_b200")
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)


def _cp(rng, dims, r, sparse=False):
    if sparse:
        fs = [sp.random_array((d, r), density=0.6, rng=rng, format="csc") + sp.eye_array(d, r)
              for d in dims]
    else:
        fs = [rng.standard_normal((d, r)) for d in dims]
    return ids.CpTensor(rng.random(r) + 0.5, fs)


def _dense(x):
    return x.to_dense()


# ---------------------------------------------------------------- hash ------
def test_square_surjective_is_a_permutation_and_wide_is_rejected():
    for n in (1, 4, 17, 300):
        op = ids.CountSketchOp(n, n, seed=n, surjective=True)
        assert sorted(op.bucket.tolist()) == list(range(n))
    with pytest.raises(ValueError):
        ids.CountSketchOp(6, 11, seed=0, surjective=True)
    with pytest.raises(ValueError):
        ids.CountSketchOp(0, 3, seed=0)


def test_standard_buckets_uniform_chi_square():
    counts = np.zeros(64)
    for trial in range(300):
        counts += np.bincount(ids.CountSketchOp(5000, 64, seed=trial).bucket, minlength=64)
    assert stats.chisquare(counts).pvalue > 0.001


def test_operator_mass_and_surjective_rank():
    op = ids.CountSketchOp(91, 13, seed=4)
    assert np.sum(op.materialize() ** 2) == 91.0  # one +-1 per column
    op = ids.CountSketchOp(70, 15, seed=8, surjective=True)
    assert np.linalg.matrix_rank(op.materialize()) == 15


def test_tensorsketch_needs_modes():
    with pytest.raises(ValueError):
        ids.TensorSketchOp([], 4)


def test_zero_matrix_zero_sketch():
    op = ids.CountSketchOp(50, 7, seed=1, surjective=True)
    assert np.array_equal(op.apply(np.zeros((50, 3))), np.zeros((7, 3)))
    assert np.array_equal(op.apply(sp.csr_array((50, 3))), np.zeros((7, 3)))


# ---------------------------------------------------------------- CP tensor -
def test_cp_normalization_sign_and_zero_columns():
    x = ids.CpTensor([3.0], [np.array([[6.0], [8.0]]), np.array([[0.0], [0.5]])])
    assert x.weights[0] == pytest.approx(3.0 * 10.0 * 0.5)
    for f in x.factors:
        assert np.linalg.norm(f[:, 0]) == pytest.approx(1.0, abs=1e-12)
    x = ids.CpTensor([-2.0], [np.ones((3, 1)), np.ones((2, 1))])
    assert x.weights[0] > 0.0 and np.allclose(x.to_dense(), -2.0 * np.ones((3, 2)))
    x = ids.CpTensor([1.0, 4.0], [np.array([[0.0, 2.0], [0.0, 0.0]]), np.eye(2)])
    assert list(x.zero_columns) == [0] and x.weights[0] == 0.0
    x = ids.CpTensor([1.0, 4.0], [sp.csc_array(np.array([[0.0, 2.0], [0.0, 0.0]])), np.eye(2)])
    assert list(x.zero_columns) == [0] and x.weights[0] == 0.0
    with pytest.raises(ValueError):
        ids.CpTensor([1.0], [np.ones((2, 1)), np.ones((2, 3))])


def test_gram_hadamard_properties():
    x = ids.CpTensor([4.0], [np.ones((3, 1)), np.ones((5, 1))])
    g = ids.gram_hadamard(x)
    assert g.shape == (1, 1) and g[0, 0] == pytest.approx(x.weights[0] ** 2, rel=1e-14)
    rng = np.random.default_rng(20)
    q1 = np.linalg.qr(rng.standard_normal((7, 4)))[0]
    q2 = np.linalg.qr(rng.standard_normal((6, 4)))[0]
    lam = np.array([4.0, 3.0, 2.0, 1.0])
    assert np.abs(ids.gram_hadamard(ids.CpTensor(lam, [q1, q2])) - np.diag(lam ** 2)).max() <= 1e-12
    for sparse in (False, True):
        x = _cp(rng, (4, 5, 3), 4, sparse=sparse)
        m = khatri_rao([f.toarray() if sp.issparse(f) else f for f in x.factors]) * x.weights
        assert np.abs(ids.gram_hadamard(x) - m.T @ m).max() <= 1e-12
    for _ in range(5):
        g = ids.gram_hadamard(_cp(rng, (3, 4, 5), 6))
        assert np.linalg.eigvalsh(g).min() >= -1e-10 * np.trace(g)


def test_cp_norms_against_dense():
    rng = np.random.default_rng(21)
    x = ids.CpTensor([7.0], [np.ones((4, 1)) / 2.0, np.ones((9, 1)) / 3.0])
    assert ids.cp_norm(x) == pytest.approx(7.0, rel=1e-12)
    x = _cp(rng, (3, 4, 3), 3)
    assert ids.cp_diff_norm(x, x) <= 1e-7 * ids.cp_norm(x)
    dense = np.linalg.norm(_dense(x))
    assert abs(ids.cp_norm(x) - dense) <= 1e-10 * dense
    y = _cp(rng, (3, 4, 3), 2)
    d = np.linalg.norm(_dense(x) - _dense(y))
    assert abs(ids.cp_diff_norm(x, y) - d) <= 1e-9 * d
    xs = _cp(rng, (3, 4, 3), 3, sparse=True)
    d = np.linalg.norm(_dense(xs) - _dense(y))
    assert abs(ids.cp_diff_norm(xs, y) - d) <= 1e-9 * d
    with pytest.raises(ValueError):
        ids.cp_diff_norm(_cp(rng, (3, 3), 2), _cp(rng, (3, 5), 2))


def test_degenerate_tensor_sketch_pads_zero_weights():
    base = np.array([[0.28], [0.96]])
    x = ids.CpTensor([1.0, 1.0], [np.hstack([base, base])] * 3)
    res = ids.tensorsketch_id(x, 2, sketch_dim=4, seed=6)
    assert res.rank_deficient and res.numerical_rank == 1
    assert np.all(res.reduced.weights[res.numerical_rank:] == 0.0)
    want, _ = oracle.tensorsketch_id(x.weights, x.factors, 2, 4, seed=6)
    assert want.rank_deficient and want.numerical_rank == 1


# ---------------------------------------------------------------- estimator -
def test_estimator_known_spectrum_and_zero():
    ap, adj = ids.matrix_operator(np.diag([5.0, 2.0, 0.25, 0.1]))
    est = ids.est_spectral_norm(ap, adj, cols=4, iters=25, probes=3, seed=3)
    assert 4.999 <= est.value <= 5.0 and est.iterations == 25 and est.probes == 3
    ap, adj = ids.matrix_operator(np.zeros((6, 4)))
    assert ids.est_spectral_norm(ap, adj, cols=4, seed=2).value == 0.0


def test_estimator_never_exceeds_and_is_monotone():
    rng = np.random.default_rng(22)
    for trial in range(25):
        a = rng.standard_normal((int(rng.integers(4, 50)), int(rng.integers(4, 50))))
        ap, adj = ids.matrix_operator(a)
        v = ids.est_spectral_norm(ap, adj, cols=a.shape[1], iters=6, seed=trial).value
        assert v <= np.linalg.norm(a, 2) + 1e-10
    a = rng.standard_normal((40, 25))
    ap, adj = ids.matrix_operator(a)
    prev = -np.inf
    for iters in (1, 3, 6, 12):
        v = ids.est_spectral_norm(ap, adj, cols=25, iters=iters, seed=9).value
        assert v >= prev - 1e-12
        prev = v


def test_residual_operator_matches_explicit_residual():
    rng = np.random.default_rng(23)
    for a in (sp.random_array((80, 30), density=0.25, rng=rng, format="csc"),
              rng.standard_normal((70, 8)) @ rng.standard_normal((8, 30))):
        d = ids.countsketch_id(a, 8, seed=4)
        dense = a.toarray() if sp.issparse(a) else a
        resid = dense[:, d.cols] @ d.coeffs - dense
        ap, adj = ids.id_residual_operator(a, d)
        x, y = rng.standard_normal(30), rng.standard_normal(dense.shape[0])
        assert np.abs(ap(x).cpu().numpy() - resid @ x).max() <= 1e-10
        assert np.abs(adj(y).cpu().numpy() - resid.T @ y).max() <= 1e-10
        est = ids.est_spectral_norm(ap, adj, cols=30, iters=15, probes=3, seed=5).value
        true = np.linalg.norm(resid, 2)
        assert est <= true + 1e-10 and est >= true / 2.0
        assert relerr_fro(np.array([est]), np.array([true])) <= 0.5


# ---------------------------------------------------------------- I/O --------
def test_matrix_market_to_device_feeds_the_path(tmp_path):
    from scipy.io import mmwrite

    rng = np.random.default_rng(24)
    a = sp.random_array((4000, 150), density=0.03, rng=rng, format="csc")
    p = tmp_path / "a.mtx"
    mmwrite(p, a, precision=17)
    host = ids.read_matrix_market(p)
    dev = ids.read_matrix_market_device(p)
    assert dev.kind == "csr" and dev.shape == (4000, 150)
    op = ids.CountSketchOp(4000, 30, seed=7, surjective=True)
    assert np.array_equal(op.apply(dev), op.apply(host))  # both ordered: scipy's sums
    d1 = ids.countsketch_id(host, 10, 30, seed=7)
    d2 = ids.countsketch_id(dev, 10, 30, seed=7)
    assert np.array_equal(d1.cols, d2.cols) and np.array_equal(d1.coeffs, d2.coeffs)
    w = oracle.countsketch_id(host, 10, 30, seed=7)
    assert np.array_equal(d1.cols, w.cols)
    x = rng.standard_normal((60, 7))
    mmwrite(p, x, precision=17)
    t = ids.read_matrix_market_device(p)
    assert t.is_cuda and np.array_equal(t.cpu().numpy(), x)

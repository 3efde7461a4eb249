"""The error metric on the GPU (SURVEY.md §8d parity check, §8f-3): the
reference's est_spectral_norm / id_residual_operator / matrix_operator and
cp_norm / cp_diff_norm, against golden values made by the real reference and
against the CPU oracle."""

import numpy as np
import pytest
import scipy.sparse as sp

import oracle

from conftest import relerr_fro

pytestmark = pytest.mark.gpu

ids = pytest.importorskip("paper_1901_10559_b200")
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1901_10559_b200.estimators import _DeviceMatrix  # noqa: E402

RTOL = 1e-9  # power iteration on the same starts; only summation order differs


class _Decomp:
    def __init__(self, cols, coeffs):
        self.cols, self.coeffs = cols, coeffs


def test_error_estimates_vs_reference_golden(golden):
    data, man = golden
    a = data["csid_a"]
    a_sp = sp.csr_array(
        (data["csid_sp_data"], data["csid_sp_indices"], data["csid_sp_indptr"]), shape=(3000, 120)
    )
    variants = {
        "C": np.ascontiguousarray(a),
        "F": np.asfortranarray(a),
        "cuda": torch.from_numpy(a).cuda(),
    }
    for case in man["error_estimates"]:
        want = case["value"]
        if case["case"] == "csid":
            s = case["seed"]
            assert ids.derive_seed(s, 0xE57) == case["est_seed"]
            d = _Decomp(data[f"csid{s}_cols"], data[f"csid{s}_coeffs"])
            for name, av in variants.items():
                ap, adj = ids.id_residual_operator(av, d)
                got = ids.est_spectral_norm(ap, adj, cols=120, seed=case["est_seed"])
                assert got.iterations == 10 and got.probes == 2
                assert abs(got.value - want) <= RTOL * want, (s, name, got.value, want)
        elif case["case"] == "csid_sp":
            d = _Decomp(data["csid_sp_cols"], data["csid_sp_coeffs"])
            for av in (a_sp, sp.csc_array(a_sp), a_sp.tocoo()):
                ap, adj = ids.id_residual_operator(av, d)
                got = ids.est_spectral_norm(ap, adj, cols=120, seed=case["est_seed"])
                assert abs(got.value - want) <= RTOL * want, (av.format, got.value, want)
        else:
            ap, adj = ids.matrix_operator(a)
            got = ids.est_spectral_norm(ap, adj, cols=120, iters=case["iters"],
                                        probes=case["probes"], seed=case["est_seed"])
            assert abs(got.value - want) <= RTOL * want


def test_end_to_end_trial_error_matches_oracle():
    """run_matrix_trial's metric (bench.py:123-146) on our ID vs the oracle's."""
    rng = np.random.default_rng(31)
    a = rng.standard_normal((20_000, 30)) @ rng.standard_normal((30, 400))
    a += 1e-3 * rng.standard_normal(a.shape)
    for seed in range(3):
        d = ids.countsketch_id(a, 25, 60, seed=seed)
        w = oracle.countsketch_id(a, 25, 60, seed=seed)
        assert np.array_equal(d.cols, w.cols)
        es = oracle.derive_seed(seed, 0xE57)
        ap, adj = ids.id_residual_operator(a, d)
        mine = ids.est_spectral_norm(ap, adj, cols=400, seed=es).value
        oap, oadj = oracle.id_residual_operator(a, w.cols, w.coeffs)
        ref = oracle.est_spectral_norm(oap, oadj, 400, seed=es)
        assert abs(mine - ref) <= 0.01 * ref  # within 1%
        assert abs(mine - ref) <= 1e-8 * ref


@pytest.mark.parametrize("layout", ["C", "F"])
@pytest.mark.parametrize("rows,cols", [(1, 1), (3, 9000), (9000, 3), (257, 300), (40_000, 70),
                                       (70, 40_000), (5, 20_000)])
def test_dense_gemv_vs_numpy(layout, rows, cols):
    rng = np.random.default_rng(rows * 7 + cols)
    a = rng.standard_normal((rows, cols))
    a = np.ascontiguousarray(a) if layout == "C" else np.asfortranarray(a)
    m = _DeviceMatrix(a)
    x = rng.standard_normal(cols)
    y = rng.standard_normal(rows)
    ax = m.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    aty = m.matvec(torch.from_numpy(y).cuda(), trans=True).cpu().numpy()
    assert relerr_fro(ax, a @ x) <= 1e-13
    assert relerr_fro(aty, a.T @ y) <= 1e-13
    # deterministic summation order
    again = m.matvec(torch.from_numpy(y).cuda(), trans=True).cpu().numpy()
    assert np.array_equal(aty, again)


def test_dense_gemv_strided_device_view():
    rng = np.random.default_rng(3)
    base = torch.from_numpy(rng.standard_normal((500, 64))).cuda()
    view = base[:, 5:45]  # row-major with ld 64
    m = _DeviceMatrix(view)
    x = rng.standard_normal(40)
    got = m.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert relerr_fro(got, view.cpu().numpy() @ x) <= 1e-13


@pytest.mark.parametrize("rows,cols,density", [(1, 1, 1.0), (500, 300, 0.002), (2000, 50, 0.3),
                                               (300, 3000, 0.05), (10_000, 200, 0.001)])
def test_sparse_passes_and_transpose_vs_scipy(rows, cols, density):
    rng = np.random.default_rng(rows + cols)
    a = sp.random_array((rows, cols), density=density, rng=rng, format="csr")
    x = rng.standard_normal(cols)
    y = rng.standard_normal(rows)
    for av in (a, sp.csc_array(a)):
        m = _DeviceMatrix(av)
        ax = m.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
        aty = m.matvec(torch.from_numpy(y).cuda(), trans=True).cpu().numpy()
        assert np.abs(ax - a @ x).max() <= 1e-12 * max(1.0, np.abs(a @ x).max())
        assert np.abs(aty - a.T @ y).max() <= 1e-12 * max(1.0, np.abs(a.T @ y).max())
    # the device transpose equals scipy's CSC (rows increasing within each column)
    m = _DeviceMatrix(a)
    t_indptr, t_indices, t_data = (v.cpu().numpy() for v in m.csr_t)
    csc = sp.csc_array(a)
    csc.sort_indices()
    assert np.array_equal(t_indptr, csc.indptr)
    assert np.array_equal(t_indices[:a.nnz], csc.indices)
    assert np.array_equal(t_data[:a.nnz], csc.data)


def test_estimator_argument_errors_and_host_callables():
    a = np.random.default_rng(0).standard_normal((30, 10))
    ap, adj = ids.matrix_operator(a)
    with pytest.raises(ValueError):
        ids.est_spectral_norm(ap, adj, cols=0)
    with pytest.raises(ValueError):
        ids.est_spectral_norm(ap, adj, cols=10, iters=-1)
    with pytest.raises(ValueError):
        ids.est_spectral_norm(ap, adj, cols=10, probes=0)
    # an inconsistent pair fails the adjoint test (estimators.py:60-66)
    with pytest.raises(ValueError):
        ids.est_spectral_norm(ap, lambda y: 2.0 * (a.T @ y), cols=10, seed=1)
    # plain host callables work and agree with the reference restatement
    got = ids.est_spectral_norm(lambda x: a @ x, lambda y: a.T @ y, cols=10, seed=4).value
    want = oracle.est_spectral_norm(lambda x: a @ x, lambda y: a.T @ y, 10, seed=4)
    assert abs(got - want) <= RTOL * want
    assert got <= np.linalg.norm(a, 2) * (1 + 1e-12)


def test_cp_norms_vs_reference_golden(golden):
    data, man = golden
    case = man["tensorsketch_id"][0]
    factors = [data[f"tsid_f{m}"] for m in range(len(case["dims"]))]
    x = ids.CpTensor(data["tsid_w"], factors)
    assert abs(ids.cp_norm(x) - case["cp_norm"]) <= 1e-12 * case["cp_norm"]
    res = ids.tensorsketch_id(x, case["rank"], case["sketch_dim"], seed=case["seed"])
    err = ids.cp_diff_norm(x, res.reduced)
    assert abs(err - case["cp_diff_norm"]) <= 1e-8 * case["cp_norm"]
    g = ids.gram_hadamard(x)
    assert relerr_fro(g, oracle.cp_gram(x.weights, x.factors)) <= 1e-13
    with pytest.raises(ValueError):
        ids.cp_diff_norm(x, ids.CpTensor(np.ones(2), [np.ones((3, 2))] * 3))


def test_cp_diff_norm_sparse_factors():
    rng = np.random.default_rng(15)
    fs = [sp.random_array((12, 6), density=0.4, rng=rng, format="csc") + sp.eye_array(12, 6)
          for _ in range(3)]
    x = ids.CpTensor(rng.random(6) + 0.5, fs)
    res = ids.tensorsketch_id(x, 3, seed=4)
    got = ids.cp_diff_norm(x, res.reduced)
    want = oracle.cp_diff_norm(x.weights, [f.toarray() for f in x.factors],
                               res.reduced.weights, [f.toarray() for f in res.reduced.factors])
    assert abs(got - want) <= 1e-10 * oracle.cp_norm(x.weights, [f.toarray() for f in x.factors])

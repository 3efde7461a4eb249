"""Host-side logic of the drop-in surface that runs before any device work."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1901_10559_b200 as ids
from paper_1901_10559_b200.cp_tensor import CpTensor, check_tensor_id_args
from paper_1901_10559_b200.matrix_id import check_matrix_id_args
from paper_1901_10559_b200.sketch import _seed_entropy, seed_state

import oracle


def test_seed_state_matches_numpy_default_rng():
    for seed in (0, 1, 99, 2**40 + 3):
        st, inc = seed_state(seed)
        ref = np.random.default_rng(seed).bit_generator.state["state"]
        assert (st, inc) == (ref["state"], ref["inc"])
    ss = np.random.SeedSequence([5, 2])
    assert seed_state(ss) == oracle.seed_state(5, mode=2)


def test_seed_entropy():
    assert _seed_entropy(7) == 7
    assert _seed_entropy(np.random.SeedSequence(11)) == 11
    assert isinstance(_seed_entropy(None), int)


def test_countsketch_validation_before_device():
    with pytest.raises(ValueError):
        ids.CountSketchOp(0, 3)
    with pytest.raises(ValueError):
        ids.CountSketchOp(5, 10, surjective=True)
    with pytest.raises(ValueError):
        ids.TensorSketchOp([], 4)
    with pytest.raises(ValueError):
        ids.TensorSketchOp([3, 0], 4)


def test_from_arrays_validation():
    with pytest.raises(ValueError):
        ids.CountSketchOp.from_arrays([0, 1], [1.0, 0.5])
    with pytest.raises(ValueError):
        ids.CountSketchOp.from_arrays([[0, 1]], [[1.0, 1.0]])


class _Shape:
    def __init__(self, shape):
        self.shape = shape


def test_check_matrix_id_args():
    assert check_matrix_id_args(_Shape((100, 30)), 5, None) == 15
    with pytest.raises(ValueError):
        check_matrix_id_args(_Shape((20, 10)), 5, 20)  # L >= rows
    with pytest.raises(ValueError):
        check_matrix_id_args(_Shape((20, 10)), 5, 4)  # L < k
    with pytest.raises(ValueError):
        check_matrix_id_args(_Shape((20, 10)), 11, None)  # k > cols
    with pytest.raises(ValueError):
        check_matrix_id_args(_Shape((20, 10)), 0, None)


def test_cptensor_normalization_matches_reference_rules():
    rng = np.random.default_rng(3)
    f0 = rng.standard_normal((5, 4))
    f1 = rng.standard_normal((6, 4))
    f1[:, 2] = 0.0
    w = np.array([1.0, -2.0, 3.0, 0.5])
    x = CpTensor(w, [f0, f1])
    assert np.all(x.weights >= 0)
    assert list(x.zero_columns) == [2]
    assert x.weights[2] == 0.0
    for f in x.factors:
        assert np.allclose(np.linalg.norm(f, axis=0), 1.0)
    # weights * normalized outer products reproduce the tensor
    dense = np.einsum("r,ir,jr->ij", w, f0, f1)
    assert np.allclose(x.to_dense(), dense)
    # unit columns stay bit-identical through select
    y = x.select([0, 3], x.weights[[0, 3]])
    assert np.array_equal(y.factors[0], x.factors[0][:, [0, 3]])


def test_cptensor_sparse_factors_and_errors():
    f = sp.random_array((8, 3), density=0.5, rng=np.random.default_rng(1), format="csc")
    x = CpTensor(np.ones(3), [f, np.ones((2, 3))])
    assert sp.issparse(x.factors[0])
    with pytest.raises(ValueError):
        CpTensor(np.ones(2), [np.ones((3, 3))])
    with pytest.raises(ValueError):
        CpTensor(np.ones(3), [np.ones((3, 3)), np.ones((2, 2))])
    with pytest.raises(ValueError):
        CpTensor(np.array([1.0, np.nan, 1.0]), [np.ones((3, 3))])
    with pytest.raises(ValueError):
        CpTensor(np.ones(1), [])


def test_check_tensor_id_args():
    x = CpTensor(np.ones(4), [np.random.default_rng(0).standard_normal((5, 4))] * 2)
    assert check_tensor_id_args(x, 2, None, "tensorsketch") == 12  # k + 10
    with pytest.raises(ValueError):
        check_tensor_id_args(x, 5, None, "tensorsketch")
    with pytest.raises(ValueError):
        check_tensor_id_args(x, 2, 25, "tensorsketch")
    with pytest.raises(ValueError):
        check_tensor_id_args(x, 2, 1, "tensorsketch")


def test_sparse_sketch_mode_validation():
    import paper_1901_10559_b200 as ids

    prev = ids.set_sparse_sketch_mode("stream")
    assert ids.set_sparse_sketch_mode(prev) == "stream"
    with pytest.raises(ValueError):
        ids.set_sparse_sketch_mode("fast")


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_cptensor_select_matches_full_constructor(seed):
    """select() on dense factors skips re-validation; the result must equal
    CpTensor(weights, the selected columns) bit for bit (zero columns, signs
    moved into mode 0, -0.0 and 0 weights, repeated columns)."""
    rng = np.random.default_rng(seed)
    facs = [np.asfortranarray(rng.standard_normal((50 + 7 * n, 40))) for n in range(3)]
    facs[1][:, 3] = 0.0
    x = CpTensor(rng.standard_normal(40), facs)
    cols = np.concatenate([[3, 3], rng.choice(40, 10, replace=False)])
    w = rng.standard_normal(cols.size)
    w[2], w[4] = 0.0, -0.0
    for ww in (w, np.abs(w)):
        got = x.select(cols, ww)
        want = CpTensor(ww, [f[:, cols] for f in x.factors])
        assert all(np.array_equal(a, b) for a, b in zip(got.factors, want.factors))
        assert np.array_equal(got.weights, want.weights)
        assert np.array_equal(np.signbit(got.weights), np.signbit(want.weights))
        assert np.array_equal(got.zero_columns, want.zero_columns)
        assert all(f.flags.f_contiguous for f in got.factors)
    with pytest.raises(ValueError):
        x.select(cols, np.full(cols.size, np.nan))

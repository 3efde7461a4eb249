"""Boundary shapes and input kinds of the matrix path against the oracle."""

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


def _same_id(d, w):
    assert np.array_equal(d.cols, w.cols)
    assert relerr_fro(d.coeffs, w.coeffs) <= 1e-10
    assert d.numerical_rank == w.numerical_rank and d.rank_deficient == w.rank_deficient


@pytest.mark.parametrize("rows,cols,k,L", [(50, 1, 1, 1), (12, 30, 5, 5), (21, 9, 3, 20),
                                           (2, 3, 1, 1), (300, 40, 40, 41)])
def test_boundary_shapes(rows, cols, k, L):
    rng = np.random.default_rng(rows * 100 + cols)
    a = rng.standard_normal((rows, cols))
    for surj in (True, False):
        d = ids.countsketch_id(a, k, L, seed=rows, surjective=surj)
        w = oracle.countsketch_id(a, k, L, seed=rows, surjective=surj)
        assert np.array_equal(d.cols[:w.numerical_rank], w.cols[:w.numerical_rank])
        if not w.rank_deficient:
            _same_id(d, w)


def test_input_kinds_agree():
    rng = np.random.default_rng(50)
    base = rng.standard_normal((400, 8)) @ rng.standard_normal((8, 60))
    want = oracle.countsketch_id(base, 8, 24, seed=2)
    kinds = {
        "C": base,
        "F": np.asfortranarray(base),
        "strided numpy view": np.hstack([base, base])[:, :60],
        "float32": base.astype(np.float32),
        "int": np.round(base * 1000).astype(np.int64),
        "cuda": torch.from_numpy(base).cuda(),
        "cuda padded rows": torch.nn.functional.pad(torch.from_numpy(base), (0, 5)).cuda()[:, :60],
        "cuda transposed": torch.from_numpy(np.ascontiguousarray(base.T)).cuda().t(),
        "cuda padded columns": torch.nn.functional.pad(
            torch.from_numpy(np.ascontiguousarray(base.T)), (0, 7)).cuda()[:, :400].t(),
    }
    for name, a in kinds.items():
        d = ids.countsketch_id(a, 8, 24, seed=2)
        if name in ("float32", "int"):
            w = oracle.countsketch_id(np.asarray(a, dtype=np.float64), 8, 24, seed=2)
            _same_id(d, w)
        else:
            _same_id(d, want)
    # sparse formats: CSR (int32 and int64 indptr), CSC, COO with duplicates
    s = sp.random_array((500, 70), density=0.05, rng=rng, format="csr")
    w = oracle.countsketch_id(sp.csc_array(s), 6, 20, seed=3)
    s64 = sp.csr_array((s.data, s.indices.astype(np.int64), s.indptr.astype(np.int64)), shape=s.shape)
    coo = s.tocoo()
    dup = sp.coo_array((np.concatenate([coo.data / 2, coo.data / 2]),
                        (np.concatenate([coo.row, coo.row]), np.concatenate([coo.col, coo.col]))),
                       shape=s.shape)
    for a in (s, s64, sp.csc_array(s), dup):
        _same_id(ids.countsketch_id(a, 6, 20, seed=3), w)


def test_argument_errors():
    a = np.ones((10, 4))
    for bad in (dict(rank=0), dict(rank=5), dict(rank=2, sketch_dim=1), dict(rank=2, sketch_dim=10)):
        with pytest.raises(ValueError):
            ids.countsketch_id(a, **bad)
    with pytest.raises(ValueError):
        ids.countsketch_id(np.ones(10), 1)
    with pytest.raises(ValueError):
        ids.countsketch_id(np.ones((0, 3)), 1)
    bad = sp.eye_array(10, 3, format="csr") * 1.0
    bad.data[0] = np.inf
    with pytest.raises(ValueError):
        ids.countsketch_id(bad, 1, 2)


def test_rank_tol_zero_singular_triangle_raises():
    """rank_tol = 0 leaves an exactly zero R11 diagonal unfloored; the
    reference's triangular_solve then raises SingularTriangleError
    (matrix_id.py:68-80, linalg.py:141-144) -- so does the device solve."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal((60, 3)) @ rng.standard_normal((3, 9))
    a[:, 3:] = 0.0  # rank 3 with 6 exactly zero columns: pivots 4.. have zero norm
    with pytest.raises(ids.SingularTriangleError, match="index 3"):
        ids.matrix_id(a, 5, rank_tol=0.0)
    d = ids.matrix_id(a, 5)  # default rank_tol floors the zero diagonal instead
    assert d.rank_deficient and np.all(np.isfinite(d.coeffs))


@pytest.mark.parametrize("I,L,surj,pre", [(5000, 37, True, 0), (3001, 64, False, 2),
                                          (999, 5, True, 3)])
def test_generator_seed_draws_and_advances_like_numpy(I, L, surj, pre):
    """default_rng(gen) draws from gen itself (reference sketch.py:77): same
    bucket / sign as numpy's draws, and gen left where numpy leaves it."""
    g1 = np.random.default_rng(1234)
    g2 = np.random.default_rng(1234)
    for g in (g1, g2):  # an even number of 32-bit draws already taken
        g.integers(0, 7, size=2 * pre, dtype=np.int32)
    rng = np.random.default_rng(g2)
    if surj:
        tail = rng.integers(0, L, size=I - L)
        want_b = rng.permutation(np.concatenate([np.arange(L, dtype=np.int64), tail]))
    else:
        want_b = rng.integers(0, L, size=I)
    want_s = rng.integers(0, 2, size=I).astype(np.float64) * 2.0 - 1.0
    op = ids.CountSketchOp(I, L, seed=g1, surjective=surj)
    assert np.array_equal(op.bucket, want_b) and np.array_equal(op.sign, want_s)
    assert np.array_equal(g1.integers(0, 2**31, size=9), g2.integers(0, 2**31, size=9))
    assert g1.bit_generator.state == g2.bit_generator.state


def test_results_survive_later_calls():
    """Coefficients are views of the call's own pinned result buffer: later
    calls (which reuse freed pinned blocks) must not change earlier results."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal((3000, 400))
    r1 = ids.countsketch_id(a, 10, 60, seed=1)
    keep = (r1.coeffs.copy(), r1.cols.copy())
    from paper_1901_10559_b200.matrix_id import countsketch_id_trials

    trials = countsketch_id_trials(a, 10, 60, seeds=[5, 6, 7])
    keep_t = [(t.coeffs.copy(), t.cols.copy()) for t in trials]
    for s in range(8, 14):
        ids.countsketch_id(a, 10, 60, seed=s)
        countsketch_id_trials(a, 10, 60, seeds=[s, s + 1])
    assert np.array_equal(r1.coeffs, keep[0]) and np.array_equal(r1.cols, keep[1])
    for t, (c, j) in zip(trials, keep_t):
        assert np.array_equal(t.coeffs, c) and np.array_equal(t.cols, j)
    assert r1.coeffs.flags.c_contiguous and r1.coeffs.flags.writeable

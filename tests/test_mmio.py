"""Matrix Market / CP-directory I/O: the native parser
against scipy.io.mmread -- the call behind the reference's read_matrix_market
(mmio.py:23-28) -- on files written the way the reference writes them.  Host
code only: runs without a GPU."""

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.io import mmread, mmwrite

from paper_1901_10559_b200 import mmio


def _ref_read(path):
    """reference mmio.read_matrix_market: as_csc / as_dense of scipy's mmread."""
    a = mmread(path, spmatrix=False)
    if sp.issparse(a):
        out = sp.csc_array(a, dtype=np.float64)
        out.sum_duplicates()
        out.eliminate_zeros()
        out.sort_indices()
        return out
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _same(a, b):
    if sp.issparse(a):
        assert sp.issparse(b) and a.shape == b.shape
        assert np.array_equal(a.indptr, b.indptr)
        assert np.array_equal(a.indices, b.indices)
        assert np.array_equal(a.data, b.data)  # correctly rounded parse: bit-identical
    else:
        assert not sp.issparse(b) and a.shape == b.shape
        assert np.array_equal(a, b) and a.flags.f_contiguous


@pytest.mark.parametrize("shape,density", [((1, 1), 1.0), ((40, 25), 0.1), ((500, 300), 0.02),
                                           ((3000, 7), 0.3)])
def test_coordinate_general_matches_scipy(tmp_path, shape, density):
    rng = np.random.default_rng(shape[0])
    m = sp.random_array(shape, density=density, rng=rng, format="csc")
    m.data = rng.standard_normal(m.nnz) * 10.0 ** rng.integers(-300, 300, m.nnz)
    p = tmp_path / "m.mtx"
    mmwrite(p, m, precision=17, symmetry="general")
    _same(mmio.read_matrix_market(p), _ref_read(p))


def test_symmetric_skew_pattern_integer(tmp_path):
    rng = np.random.default_rng(1)
    s = sp.random_array((30, 30), density=0.2, rng=rng).toarray()
    sym = s + s.T
    skew = s - s.T
    for mat, kw in ((sp.coo_array(sym), {"symmetry": "symmetric"}),
                    (sp.coo_array(skew), {"symmetry": "skew-symmetric"}),
                    (sp.coo_array((sym != 0).astype(float)), {"field": "pattern"}),
                    (sp.coo_array(np.round(10 * sym)), {"field": "integer"})):
        p = tmp_path / "s.mtx"
        mmwrite(p, mat, **kw)
        _same(mmio.read_matrix_market(p), _ref_read(p))


def test_array_format_general_and_symmetric(tmp_path):
    rng = np.random.default_rng(2)
    a = rng.standard_normal((17, 9))
    p = tmp_path / "a.mtx"
    mmwrite(p, a, precision=17)
    _same(mmio.read_matrix_market(p), _ref_read(p))
    s = rng.standard_normal((6, 6))
    mmwrite(p, s + s.T, symmetry="symmetric", precision=17)
    _same(mmio.read_matrix_market(p), _ref_read(p))
    mmwrite(p, s - s.T, symmetry="skew-symmetric", precision=17)
    _same(mmio.read_matrix_market(p), _ref_read(p))


def test_comments_crlf_case_and_duplicates(tmp_path):
    p = tmp_path / "c.mtx"
    p.write_bytes(b"%%MatrixMarket MATRIX Coordinate Real General\r\n% a comment\r\n\r\n"
                  b"3 4 5\r\n1 1 1.5\r\n3 4 -2e-3\r\n% inside\r\n1 1 0.25\r\n2 2 0\r\n"
                  b"  3   1   7\r\n")
    got = mmio.read_matrix_market(p)
    want = np.zeros((3, 4))
    want[0, 0], want[2, 3], want[2, 0] = 1.75, -2e-3, 7.0
    assert np.array_equal(got.toarray(), want)
    assert got.nnz == 3  # duplicates summed, the explicit zero removed


def test_errors(tmp_path):
    p = tmp_path / "bad.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n")
    with pytest.raises(ValueError):
        mmio.read_matrix_market(p)  # fewer entries than the size line says
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
    with pytest.raises(ValueError):
        mmio.read_matrix_market(p)  # row out of range
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 nan\n")
    with pytest.raises(ValueError):
        mmio.read_matrix_market(p)  # non-finite (linalg.py:51-52)
    p.write_text("not a matrix market file\n")
    with pytest.raises(ValueError):
        mmio.read_matrix_market(p)
    with pytest.raises(ValueError):
        mmio.read_matrix_market(tmp_path / "missing.mtx")


def test_write_read_roundtrip_exact(tmp_path):
    rng = np.random.default_rng(3)
    m = sp.random_array((50, 20), density=0.15, rng=rng, format="csr")
    p = tmp_path / "w.mtx"
    mmio.write_matrix_market(p, m)
    got = mmio.read_matrix_market(p)
    assert np.array_equal(got.toarray(), m.toarray())
    a = rng.standard_normal((8, 5))
    mmio.write_matrix_market(p, a)
    assert np.array_equal(mmio.read_matrix_market(p), a)


def test_cp_dir_roundtrip(tmp_path):
    from paper_1901_10559_b200.cp_tensor import CpTensor

    rng = np.random.default_rng(4)
    x = CpTensor(rng.random(5) + 0.5, [rng.standard_normal((d, 5)) for d in (4, 6, 3)])
    mmio.save_cp_dir(tmp_path / "cp", x)
    y = mmio.load_cp_dir(tmp_path / "cp")
    assert np.array_equal(y.weights, x.weights)
    for a, b in zip(x.factors, y.factors):
        assert np.array_equal(a, b)
    xs = CpTensor(np.ones(3), [sp.random_array((7, 3), density=0.5, rng=rng, format="csc")
                               + sp.eye_array(7, 3) for _ in range(2)])
    mmio.save_cp_dir(tmp_path / "cps", xs)
    ys = mmio.load_cp_dir(tmp_path / "cps")
    assert np.allclose(ys.weights, xs.weights, rtol=1e-15)
    (tmp_path / "cp" / "meta.json").write_text('{"n_modes": 3, "rank": 4, "mode_dims": [4, 6, 3]}')
    with pytest.raises(ValueError):
        mmio.load_cp_dir(tmp_path / "cp")

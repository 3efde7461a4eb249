"""Streaming CSR CountSketch (flags without ORDERED/DETERMINISTIC): one pass
over A in storage order with fp64 L2 reductions.  Checked against the oracle
(reference sketch.py:116-122, scipy CSR product) within the north_star
tolerance, on the shapes that stress its tiling: empty and ragged rows, rows
longer than a tile, tile-boundary nnz counts, int32/int64 row pointers,
offset row pointers, row shards accumulated into one Y."""

import zlib

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

from paper_1901_10559_b200._inputs import SparseOperand  # noqa: E402
from paper_1901_10559_b200._native import (  # noqa: E402
    IDS_FLAG_DETERMINISTIC,
    IDS_FLAG_ORDERED,
)

TILE = 2048
# summation-order rounding only: far inside north_star's 1e-10
TOL = 1e-13


def _operand(a, idx_dtype=torch.int64, offset=0):
    """Device CSR operand; `offset` shifts every row pointer (a view into a
    larger entry array, as a row slice of a bigger CSR would be)."""
    a = sp.csr_array(a)
    indptr = torch.from_numpy(a.indptr.astype(np.int64) + offset).to(idx_dtype).cuda()
    pad_i = np.zeros(offset, np.int32)
    pad_v = np.full(offset, np.nan)  # never read
    indices = torch.from_numpy(np.concatenate([pad_i, a.indices.astype(np.int32)])).cuda()
    data = torch.from_numpy(np.concatenate([pad_v, a.data.astype(np.float64)])).cuda()
    return SparseOperand("csr", indptr, indices, data, a.shape[0], a.shape[1], a.nnz)


def _sketch(op, operand, flags=0):
    return op.apply_device(operand, flags=flags).t().cpu().numpy()


def _ragged(rng, rows, cols, lens):
    indptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    indices = np.concatenate(
        [np.sort(rng.choice(cols, size=k, replace=False)) for k in lens]
    ).astype(np.int32) if indptr[-1] else np.zeros(0, np.int32)
    data = rng.standard_normal(int(indptr[-1]))
    return sp.csr_array((data, indices, indptr), shape=(rows, cols))


CASES = {
    "single": lambda rng: sp.csr_array(np.array([[2.5]])),
    "one_row_long": lambda rng: _ragged(rng, 1, 30_000, [25_000]),
    "long_row_between_empties": lambda rng: _ragged(rng, 5, 20_000, [0, 3, 19_999, 0, 7]),
    "mostly_empty_rows": lambda rng: _ragged(
        rng, 100_000, 50, np.where(rng.random(100_000) < 0.002, rng.integers(1, 20, 100_000), 0)),
    "trailing_empty_rows": lambda rng: _ragged(rng, 3000, 40, [5] * 1000 + [0] * 2000),
    "tile_exact": lambda rng: _ragged(rng, 2 * TILE // 8, 64, [8] * (2 * TILE // 8)),
    "tile_plus_one": lambda rng: _ragged(rng, 2 * TILE // 8 + 1, 64, [8] * (2 * TILE // 8) + [1]),
    "tile_minus_one": lambda rng: _ragged(rng, TILE // 8, 64, [8] * (TILE // 8 - 1) + [7]),
    "ragged": lambda rng: _ragged(rng, 4000, 700, rng.integers(0, 300, 4000)),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("idx_dtype", [torch.int64, torch.int32])
def test_stream_matches_oracle(name, idx_dtype):
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    a = CASES[name](rng)
    L = min(a.shape[0], 37) if a.shape[0] > 1 else 1
    op = ids.CountSketchOp(a.shape[0], L, seed=5, surjective=True)
    want = oracle.cs_apply(op.bucket, op.sign, L, a)
    got = _sketch(op, _operand(a, idx_dtype))
    assert relerr_fro(got, want) <= TOL, name
    # ordered mode stays bit-exact on the same operand
    assert np.array_equal(_sketch(op, _operand(a, idx_dtype), IDS_FLAG_ORDERED), want)


def test_stream_offset_row_pointers():
    rng = np.random.default_rng(1)
    a = _ragged(rng, 3000, 300, rng.integers(0, 40, 3000))
    op = ids.CountSketchOp(3000, 50, seed=2, surjective=True)
    want = oracle.cs_apply(op.bucket, op.sign, 50, a)
    for off in (1, 3, 2047, 5000):
        got = _sketch(op, _operand(a, offset=off))
        assert relerr_fro(got, want) <= TOL, off


def test_stream_empty_matrix_gives_zero():
    a = sp.csr_array((50, 7))
    op = ids.CountSketchOp(50, 5, seed=1, surjective=True)
    assert not _sketch(op, _operand(a)).any()


def test_stream_row_shards_accumulate():
    """Row blocks sketched separately (row0 offsets into the global hash,
    accumulate into one Y) equal the one-shot sketch -- the per-rank step of
    the row-sharded path."""
    rng = np.random.default_rng(4)
    a = _ragged(rng, 9000, 500, rng.integers(0, 30, 9000))
    op = ids.CountSketchOp(9000, 60, seed=8, surjective=True)
    want = oracle.cs_apply(op.bucket, op.sign, 60, a)
    y = torch.zeros((500, 60), dtype=torch.float64, device="cuda")
    for r0, r1 in [(0, 1), (1, 4000), (4000, 4001), (4001, 9000)]:
        op.sketch_into(_operand(a[r0:r1]), y, row0=r0, accumulate=True, flags=0)
    assert relerr_fro(y.t().cpu().numpy(), want) <= TOL


def test_stream_nonfinite_flagged():
    a = sp.csr_array(np.array([[1.0, 0.0], [0.0, np.inf], [2.0, 3.0]]))
    op = ids.CountSketchOp(3, 2, seed=0, surjective=True)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    y = torch.empty((2, 2), dtype=torch.float64, device="cuda")
    op.sketch_into(_operand(a), y, flags=0, nonfinite=flag)
    assert int(flag.item()) == 1


def test_large_stream_vs_deterministic_and_oracle():
    """Above the ordered threshold (2^24 nonzeros) countsketch_id streams;
    the segmented deterministic mode is run-to-run identical; both agree with
    each other and with the oracle's Y on a row sample."""
    g = torch.Generator(device="cuda").manual_seed(0)
    rows, cols, per, L = 2_000_000, 3000, 9, 120  # 1.8e7 nonzeros
    indptr = torch.arange(0, rows + 1, dtype=torch.int64, device="cuda") * per
    idx = torch.randint(0, cols, (rows, per), generator=g, device="cuda", dtype=torch.int64)
    idx = idx.sort(dim=1).values.to(torch.int32).reshape(-1)
    data = torch.randn(rows * per, generator=g, device="cuda", dtype=torch.float64)
    operand = SparseOperand("csr", indptr, idx, data, rows, cols, rows * per)
    op = ids.CountSketchOp(rows, L, seed=3, surjective=True)
    y_st = _sketch(op, operand, 0)
    y_d1 = _sketch(op, operand, IDS_FLAG_DETERMINISTIC)
    y_d2 = _sketch(op, operand, IDS_FLAG_DETERMINISTIC)
    assert np.array_equal(y_d1, y_d2)
    assert relerr_fro(y_st, y_d1) <= TOL
    # oracle on the leading 100k rows
    sub = 100_000
    a_sub = sp.csr_array(
        (data[: sub * per].cpu().numpy(), idx[: sub * per].cpu().numpy(),
         indptr[: sub + 1].cpu().numpy()), shape=(sub, cols))
    y_sub = torch.zeros((cols, L), dtype=torch.float64, device="cuda")
    op.sketch_into(SparseOperand("csr", indptr[: sub + 1], idx, data, sub, cols, sub * per),
                   y_sub, row0=0, accumulate=False, flags=0)
    want = oracle.cs_apply(op.bucket[:sub], op.sign[:sub], L, a_sub)
    assert relerr_fro(y_sub.t().cpu().numpy(), want) <= TOL


def test_deterministic_algorithms_select_segmented_mode():
    g = torch.Generator(device="cuda").manual_seed(1)
    rows, cols, per, L = 1_900_000, 800, 9, 64
    indptr = torch.arange(0, rows + 1, dtype=torch.int64, device="cuda") * per
    idx = torch.randint(0, cols, (rows * per,), generator=g, device="cuda", dtype=torch.int32)
    data = torch.randn(rows * per, generator=g, device="cuda", dtype=torch.float64)
    operand = SparseOperand("csr", indptr, idx, data, rows, cols, rows * per)
    op = ids.CountSketchOp(rows, L, seed=9, surjective=True)
    want = _sketch(op, operand, IDS_FLAG_DETERMINISTIC)
    prev = torch.are_deterministic_algorithms_enabled()
    torch.use_deterministic_algorithms(True)
    try:
        got = _sketch(op, operand, IDS_FLAG_ORDERED)  # large: ordered drops, deterministic kept
    finally:
        torch.use_deterministic_algorithms(prev)
    assert np.array_equal(got, want)


def test_c3_shaped_id_streamed_matches_oracle_error():
    """Planted-structure sparse ID (the C3 recipe, scaled down): columns 20..
    are random combinations of columns 0-19, so the ID through the streaming
    sketch must reconstruct A as well as the oracle's ID (within 1%)."""
    from paper_1901_10559_b200.matrix_id import countsketch_device

    rng = np.random.default_rng(7)
    rows, cols, k = 20_000, 300, 20
    base = sp.random_array((rows, k), density=0.01, rng=rng, format="csc")
    rest = sp.csc_array(base @ rng.standard_normal((k, cols - k)))
    a = sp.csr_array(sp.hstack([base, rest]))
    a = sp.csr_array(a + 1e-9 * sp.random_array((rows, cols), density=1e-3, rng=rng))
    d, _ = countsketch_device(a, k, 60, seed=4, flags=0)
    d = d.to_host("countsketch")
    w = oracle.countsketch_id(a, k, 60, seed=4)
    ad = a.toarray()
    e_got = np.linalg.norm(ad - ad[:, d.cols] @ d.coeffs) / np.linalg.norm(ad)
    e_want = np.linalg.norm(ad - ad[:, w.cols] @ w.coeffs) / np.linalg.norm(ad)
    assert e_got <= max(1.01 * e_want, 1e-12)


def test_sparse_sketch_modes_above_ordered_threshold():
    """Above ORDERED_SPARSE_MAX_NNZ: "auto" streams (one warning), "ordered"
    keeps scipy's order bit for bit, "deterministic" is run-to-run identical."""
    import warnings

    from paper_1901_10559_b200 import sketch as sk

    rng = np.random.default_rng(44)
    rows, cols, per = 2_000_000, 3000, 9  # 1.8e7 nonzeros > 2^24
    idx = np.sort(rng.integers(0, cols, size=(rows, per)), axis=1).astype(np.int32)
    a = sp.csr_array((rng.standard_normal(rows * per), idx.ravel(),
                      np.arange(0, rows * per + 1, per)), shape=(rows, cols))
    a.sum_duplicates()
    op = ids.CountSketchOp(rows, 50, seed=9, surjective=True)
    want = oracle.cs_apply(op.bucket, op.sign, 50, a)
    operand = _operand(a)
    prev = ids.set_sparse_sketch_mode("auto")
    try:
        sk._warned_stream = False
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            y = _sketch(op, operand, IDS_FLAG_ORDERED)
            _sketch(op, operand, IDS_FLAG_ORDERED)
        assert sum(issubclass(x.category, ids.NondeterministicSketchWarning) for x in w) == 1
        assert relerr_fro(y, want) <= 1e-13
        ids.set_sparse_sketch_mode("ordered")
        assert np.array_equal(_sketch(op, operand, 0), want)
        ids.set_sparse_sketch_mode("deterministic")
        y1, y2 = _sketch(op, operand, 0), _sketch(op, operand, 0)
        assert np.array_equal(y1, y2) and relerr_fro(y1, want) <= 1e-13
    finally:
        ids.set_sparse_sketch_mode(prev)

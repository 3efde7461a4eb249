"""Dense F-order (column-major) sketch: the tiled kernel (rows pre-sorted per
512-row tile by owner slot, slot-owned accumulators) against the oracle
(reference sketch.py:116-122 after as_dense's F-order copy, linalg.py:29),
bit for bit in scipy's order, on the shapes that stress its tiling."""

import numpy as np
import pytest
import torch

import oracle

from conftest import relerr_fro

pytestmark = pytest.mark.gpu

ids = pytest.importorskip("paper_1901_10559_b200")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1901_10559_b200._inputs import dense_operand  # noqa: E402
from paper_1901_10559_b200._native import IDS_FLAG_ORDERED  # noqa: E402


def _fortran_dev(a, pad_rows=0):
    """Device F-order view of a (leading dimension rows + pad_rows)."""
    rows, cols = a.shape
    buf = torch.empty((cols, rows + pad_rows), dtype=torch.float64, device="cuda")
    buf[:, :rows] = torch.from_numpy(np.ascontiguousarray(a.T)).cuda()
    return buf[:, :rows].t()


@pytest.mark.parametrize("rows,cols,L", [
    (512, 8, 37), (513, 8, 37), (1, 3, 1), (1000, 5, 128), (3000, 333, 100),
    (5001, 17, 1000), (2049, 300, 7), (4096, 64, 33), (10240, 20, 128), (2112, 9, 97),
    (1538, 8, 64), (20480, 600, 100), (3000, 40, 200), (2500, 30, 129), (4000, 25, 300),
    (6000, 11, 512), (1024, 301, 257), (700, 2, 2)])
@pytest.mark.parametrize("pad", [0, 1])
def test_fortran_ordered_bit_exact(rows, cols, L, pad):
    rng = np.random.default_rng(rows * 7 + cols + L)
    a = rng.standard_normal((rows, cols))
    L = min(L, rows)
    op = ids.CountSketchOp(rows, L, seed=rows + L, surjective=True)
    want = oracle.cs_apply(op.bucket, op.sign, L, a)
    got = op.apply_device(dense_operand(_fortran_dev(a, pad)), flags=IDS_FLAG_ORDERED)
    assert np.array_equal(got.t().cpu().numpy(), want)


def test_fortran_segmented_and_shards():
    """flags=0 on few columns splits rows into segments (fixed-order partials);
    row shards accumulate into one Y (the per-rank step of row sharding)."""
    rng = np.random.default_rng(5)
    rows, cols, L = 40_000, 12, 64
    a = rng.standard_normal((rows, cols))
    op = ids.CountSketchOp(rows, L, seed=2, surjective=True)
    want = oracle.cs_apply(op.bucket, op.sign, L, a)
    y0 = op.apply_device(dense_operand(_fortran_dev(a)), flags=0).t().cpu().numpy()
    y1 = op.apply_device(dense_operand(_fortran_dev(a)), flags=0).t().cpu().numpy()
    assert np.array_equal(y0, y1)
    assert relerr_fro(y0, want) <= 1e-13
    y = torch.zeros((cols, L), dtype=torch.float64, device="cuda")
    for r0, r1 in [(0, 7), (7, 20_000), (20_000, 40_000)]:
        op.sketch_into(dense_operand(_fortran_dev(a[r0:r1])), y, row0=r0, accumulate=True,
                       flags=IDS_FLAG_ORDERED)
    assert relerr_fro(y.t().cpu().numpy(), want) <= 1e-13


@pytest.mark.parametrize("L", [100, 300])
def test_fortran_ordered_shards_accumulate_bit_exact(L):
    """Ordered row shards accumulated into one Y continue each entry's sum in
    increasing row order, so the result is the one-shot sum bit for bit."""
    rng = np.random.default_rng(L)
    rows, cols = 30_000, 21
    a = rng.standard_normal((rows, cols))
    op = ids.CountSketchOp(rows, L, seed=3, surjective=True)
    want = oracle.cs_apply(op.bucket, op.sign, L, a)
    y = torch.zeros((cols, L), dtype=torch.float64, device="cuda")
    for r0, r1 in [(0, 511), (511, 1537), (1537, 20_000), (20_000, 30_000)]:
        op.sketch_into(dense_operand(_fortran_dev(a[r0:r1])), y, row0=r0, accumulate=True,
                       flags=IDS_FLAG_ORDERED)
    assert np.array_equal(y.t().cpu().numpy(), want)


def test_fortran_large_sketch_dim_falls_back():
    """L beyond the tiled kernel's shared-memory accumulators uses the
    column-stream kernel; still scipy's order."""
    rng = np.random.default_rng(9)
    rows, cols, L = 6000, 9, 4000
    a = rng.standard_normal((rows, cols))
    op = ids.CountSketchOp(rows, L, seed=4, surjective=True)
    want = oracle.cs_apply(op.bucket, op.sign, L, a)
    got = op.apply_device(dense_operand(_fortran_dev(a)), flags=IDS_FLAG_ORDERED)
    assert np.array_equal(got.t().cpu().numpy(), want)


def test_fortran_c2_shape_id_matches_c_order():
    """configs[1]-shaped input in both layouts gives the same ID (same Y)."""
    from paper_1901_10559_b200.matrix_id import countsketch_device

    g = torch.Generator(device="cuda").manual_seed(0)
    rows, cols = 400_000, 700
    a = torch.randn(rows, cols, generator=g, device="cuda", dtype=torch.float64)
    d_c, y_c = countsketch_device(dense_operand(a), 20, 100, seed=6)
    d_f, y_f = countsketch_device(dense_operand(a.t().contiguous().t()), 20, 100, seed=6)
    assert torch.equal(y_c, y_f)
    assert np.array_equal(d_c.to_host("countsketch").cols, d_f.to_host("countsketch").cols)

"""The tall truncated CPQR (cpqr_kernel) against LAPACK dgeqp3
(linalg.py:97) on the sketch shapes of C4 / C5 and their neighbours: same
pivots, same numerical rank, R and P within 1e-10; exactly deficient and
zero sketches."""

import numpy as np
import pytest

import oracle

from conftest import relerr_fro

pytestmark = pytest.mark.gpu

ids = pytest.importorskip("paper_1901_10559_b200")
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1901_10559_b200.linalg import device_cpqr  # noqa: E402


def _near_dup(rng, m, n, base, pert):
    b = rng.standard_normal((m, base))
    idx = rng.integers(0, base, size=n)
    idx[:base] = np.arange(base)
    return b[:, idx] + pert * rng.standard_normal((m, n))


def _cpqr(y, k):
    t = torch.from_numpy(np.ascontiguousarray(y.T)).cuda()
    f = device_cpqr(t, y.shape[0], y.shape[1], k)
    return f.perm.cpu().numpy(), f.rtop.cpu().numpy(), int(f.numerical_rank.item())


@pytest.mark.parametrize("m,n,k,base,pert", [
    (4096, 1000, 10, 10, 1e-3), (16384, 2000, 20, 20, 1e-4), (2048, 37, 5, 9, 1e-2),
    (1025, 300, 12, 12, 1e-3), (5000, 80, 64, 70, 1e-2), (18000, 150, 7, 7, 1e-5)])
def test_tall_cpqr_matches_lapack(m, n, k, base, pert):
    y = _near_dup(np.random.default_rng(m + n + k), m, n, base, pert)
    p1, r1, nr1 = _cpqr(y, k)
    want = oracle.cpqr(y, k)
    assert np.array_equal(p1[:k], want.perm[:k])
    assert nr1 == want.numerical_rank
    assert relerr_fro(np.abs(r1[:, :k]), np.abs(want.r[:, :k])) <= 1e-10
    d = ids.matrix_id(y, k)
    w = oracle.matrix_id(y, k)
    assert np.array_equal(d.cols, w.cols) and relerr_fro(d.coeffs, w.coeffs) <= 1e-10


def test_tall_cpqr_deficient_and_zero():
    rng = np.random.default_rng(2)
    y = rng.standard_normal((3000, 3)) @ rng.standard_normal((3, 40))  # exact rank 3
    p1, r1, nr1 = _cpqr(y, 8)
    want = oracle.cpqr(y, 8)
    assert nr1 == want.numerical_rank == 3
    assert np.array_equal(p1[:3], want.perm[:3])
    p1, r1, nr1 = _cpqr(np.zeros((2000, 30)), 4)
    assert nr1 == 0 and not np.any(r1)


@pytest.mark.parametrize("m,n,k", [(5001, 777, 13), (2049, 9000, 7), (16384, 300, 1), (3000, 20, 20),
                                   (200, 10_000, 20), (333, 5000, 9), (1024, 18_000, 5)])
def test_column_owner_kernel_vs_segment_units_and_dgeqp3(m, n, k, monkeypatch):
    """The column-owning CPQR (v in shared memory, two grid barriers per
    step, L2-pinned leading segments; 256-row units for short wide sketches
    like C3's 200 x 10000) and the segment-unit kernel agree with LAPACK's
    pivots (odd m: the bulk copy of the residual rounds up)."""
    from paper_1901_10559_b200.linalg import device_cpqr

    rng = np.random.default_rng(m + n + k)
    base = rng.standard_normal((m, min(n, 12)))
    y = base @ rng.standard_normal((min(n, 12), n)) + 1e-3 * rng.standard_normal((m, n))
    yt = torch.from_numpy(np.ascontiguousarray(y.T)).cuda()
    a = device_cpqr(yt, m, n, k)
    monkeypatch.setenv("IDS_CPQR_SEGMENT_UNITS", "1")
    b = device_cpqr(yt, m, n, k)
    want = oracle.cpqr(y, k)
    assert np.array_equal(a.perm[:k].cpu().numpy(), want.perm[:k])
    assert np.array_equal(b.perm[:k].cpu().numpy(), want.perm[:k])
    ra, rb = a.rtop.cpu().numpy(), b.rtop.cpu().numpy()
    assert np.abs(ra - rb).max() <= 1e-11 * np.abs(rb).max()

"""The short-wide truncated CPQR (cpqr_wide_kernel: column slices resident in
shared memory, one grid barrier per step) against LAPACK dgeqp3
(linalg.py:97) and, bit for bit, against the segment-unit kernel whose
arithmetic it repeats (C3's 200 x 10000 sketch and its neighbours)."""

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


def _low_rank(rng, m, n, r, noise):
    base = rng.standard_normal((m, min(n, r)))
    return base @ rng.standard_normal((min(n, r), n)) + noise * rng.standard_normal((m, n))


def _run(y, k, ld=None, colnorm2=None, want_q=False):
    m, n = y.shape
    ld = m if ld is None else ld
    buf = np.zeros((n, ld))
    buf[:, :m] = y.T
    t = torch.from_numpy(buf).cuda().reshape(-1)
    f = device_cpqr(t, m, n, k, ld=ld, colnorm2=colnorm2, want_q=want_q)
    torch.cuda.synchronize()
    return f


@pytest.mark.parametrize("m,n,k,r,noise", [
    (200, 10_000, 20, 20, 1e-2),   # C3's sketch shape
    (200, 10_000, 20, 12, 1e-3),
    (333, 5000, 9, 12, 1e-3),
    (100, 2000, 20, 20, 1e-2),     # C2's
    (40, 1000, 10, 10, 1e-2),      # C1's
    (97, 257, 31, 40, 1e-4),
    (1, 300, 1, 1, 0.0),
    (64, 4096, 64, 80, 1e-2),
    (700, 9000, 5, 5, 1e-6),
])
def test_wide_cpqr_matches_lapack_and_segment_kernel(m, n, k, r, noise, monkeypatch):
    rng = np.random.default_rng(m * 7 + n + k)
    y = _low_rank(rng, m, n, r, noise)
    a = _run(y, k)
    want = oracle.cpqr(y, k)
    assert np.array_equal(a.perm[:k].cpu().numpy(), want.perm[:k])
    assert int(a.numerical_rank.item()) == want.numerical_rank
    ra = a.rtop.cpu().numpy()
    assert relerr_fro(np.abs(ra[:, :k]), np.abs(want.r[:, :k])) <= 1e-10
    # the segment-unit kernel runs the same operations in the same order
    monkeypatch.setenv("IDS_CPQR_NO_WIDE", "1")
    monkeypatch.setenv("IDS_CPQR_SEGMENT_UNITS", "1")
    if m * n * 8 > 16 * 200 * 1024:  # too large for the one-cluster kernel
        b = _run(y, k)
        assert np.array_equal(a.perm.cpu().numpy(), b.perm.cpu().numpy())
        assert np.array_equal(ra, b.rtop.cpu().numpy())


def test_wide_cpqr_leading_dimension_norms_and_q():
    rng = np.random.default_rng(5)
    m, n, k = 150, 3000, 12
    y = _low_rank(rng, m, n, 15, 1e-3)
    want = oracle.cpqr(y, k)
    a = _run(y, k, ld=161, want_q=True)
    assert np.array_equal(a.perm[:k].cpu().numpy(), want.perm[:k])
    q = a.q.cpu().numpy().T
    assert np.abs(q.T @ q - np.eye(k)).max() <= 1e-12
    assert relerr_fro(np.abs(q), np.abs(want.q)) <= 1e-9
    n2 = torch.from_numpy((y * y).sum(axis=0)).cuda()
    b = _run(y, k, colnorm2=n2)
    assert np.array_equal(b.perm[:k].cpu().numpy(), want.perm[:k])


def test_wide_cpqr_deficient_and_zero():
    rng = np.random.default_rng(2)
    y = rng.standard_normal((300, 3)) @ rng.standard_normal((3, 2000))  # exact rank 3
    a = _run(y, 8)
    want = oracle.cpqr(y, 8)
    assert int(a.numerical_rank.item()) == want.numerical_rank == 3
    assert np.array_equal(a.perm[:3].cpu().numpy(), want.perm[:3])
    z = _run(np.zeros((120, 900)), 4)
    assert int(z.numerical_rank.item()) == 0 and not np.any(z.rtop.cpu().numpy())
    assert sorted(z.perm.cpu().numpy()) == list(range(900))


def test_wide_cpqr_id_matches_reference_at_c3_shape():
    rng = np.random.default_rng(11)
    y = _low_rank(rng, 200, 10_000, 20, 1e-2)
    d = ids.matrix_id(y, 20)
    w = oracle.matrix_id(y, 20)
    assert np.array_equal(d.cols, w.cols)
    assert relerr_fro(d.coeffs, w.coeffs) <= 1e-10

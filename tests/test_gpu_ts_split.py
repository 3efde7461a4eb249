"""Split-spectrum TensorSketch kernel (ids_tensorsketch_split_f64: two-CTA
clusters, folded CountSketch, running spectrum in TMEM) against the
one-CTA-per-term kernel, the CPU oracle (reference sketch.py:156-186) and
its plan's layout; run-to-run identity; the chunked-plan fallbacks."""

import ctypes

import numpy as np
import pytest

import oracle

from conftest import relerr_fro

pytestmark = pytest.mark.gpu

ids = pytest.importorskip("paper_1901_10559_b200")
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1901_10559_b200 import tensorsketch as tsmod  # noqa: E402
from paper_1901_10559_b200._native import call, query  # noqa: E402


def _factors(rng, dims, r):
    return [torch.from_numpy(rng.standard_normal((d, r))).cuda() for d in dims]


def _both(op, fac, w, monkeypatch):
    y, nrm = op.apply_device(fac, w, norms=True)
    monkeypatch.setattr(tsmod, "USE_SPLIT", False)
    y_old, nrm_old = op.apply_device(fac, w, norms=True)
    monkeypatch.setattr(tsmod, "USE_SPLIT", True)
    return y, nrm, y_old, nrm_old


@pytest.mark.parametrize("dims,L,r", [
    ([1000] * 3, 4096, 333),            # C4 modes
    ([10_000] * 4, 16384, 301),         # C5 modes
    ([5000, 3000, 777], 8192, 65),      # L = 8192
    ([20_000, 9000], 16384, 40),        # a mode above the single-CTA planner (chunked plan)
    ([12_000, 12_000], 4096, 30),       # later rows exceed the tail buffer: fixed chunks
    ([7, 3, 5], 4096, 3),               # short modes, fewer terms than clusters
    ([4096], 4096, 9),                  # one mode
    ([50] * 8, 4096, 17),               # eight modes
])
def test_split_matches_one_cta_kernel_and_oracle(dims, L, r, monkeypatch):
    rng = np.random.default_rng(sum(dims) + L + r)
    fac = _factors(rng, dims, r)
    w = torch.from_numpy(rng.random(r) + 0.5).cuda()
    op = ids.TensorSketchOp(dims, L, seed=5)
    assert tsmod.uses_split_kernel(len(dims), L)
    y, nrm, y_old, nrm_old = _both(op, fac, w, monkeypatch)
    assert float((y - y_old).norm() / y_old.norm()) <= 1e-13
    assert float(((nrm - nrm_old).abs() / nrm_old).max()) <= 1e-13
    ref = (y * y).sum(dim=1)
    assert float(((nrm - ref).abs() / ref).max()) <= 1e-13
    y2, nrm2 = op.apply_device(fac, w, norms=True)  # run-to-run identical
    assert torch.equal(y, y2) and torch.equal(nrm, nrm2)
    if r <= 70:
        want = oracle.OracleTensorSketch(dims, L, seed=5).apply(
            [f.cpu().numpy() for f in fac], w.cpu().numpy())
        assert relerr_fro(y.t().cpu().numpy(), want) <= 1e-12


def test_split_strided_and_unaligned_columns(monkeypatch):
    """Factor columns with ld > rows (odd ld: columns start off 16-byte
    alignment) and no weights."""
    rng = np.random.default_rng(3)
    dims, L, r = [3001, 2999, 1000], 16384, 23
    base = [torch.from_numpy(rng.standard_normal((r, d + 3))).cuda() for d in dims]
    fac = [b[:, :d].t() for b, d in zip(base, dims)]  # col-major, ld = d + 3
    op = ids.TensorSketchOp(dims, L, seed=9)
    y, _, y_old, _ = _both(op, fac, None, monkeypatch)
    assert float((y - y_old).norm() / y_old.norm()) <= 1e-13
    want = oracle.OracleTensorSketch(dims, L, seed=9).apply([f.cpu().numpy() for f in fac], None)
    assert relerr_fro(y.t().cpu().numpy(), want) <= 1e-12


@pytest.mark.parametrize("dim,L", [(10_000, 16384), (1000, 4096), (12_000, 4096), (20_000, 16384)])
def test_split_plan_layout(dim, L):
    """The folded plan against numpy: per row the slot's buffer index,
    its signs in the even / odd half, first-row flag or tail position
    (ordered by slot, then row, inside its chunk); per chunk the tail groups."""
    op = ids.CountSketchOp(dim, L, seed=11)
    plan = op._ts_split_plan().cpu().numpy().view(np.int32)
    N2 = L // 2
    cs_fixed = L // 64 * 16
    cs = int(plan[0])
    stride = (dim + 3) & ~3
    code = plan[4:4 + dim].view(np.uint32)
    goff = ((16 + stride * 4 + 15) // 16 * 16) // 4
    ngroups_cap = max(dim // 2 + 8, -(-dim // cs_fixed) * (cs_fixed // 2))
    groups = plan[goff:goff + 2 * ngroups_cap].view(np.uint32).reshape(-1, 2)
    ngroups = plan[goff + 2 * ngroups_cap:]
    b, s = op.bucket, op.sign
    slot = b % N2

    def idx(j):
        return 2 * ((j >> 1) + ((j >> 1) >> 4)) + (j & 1)

    assert np.array_equal(code & 0x3FFF, idx(slot))
    assert np.array_equal((code >> 14) & 1, (s < 0).astype(np.uint32))
    assert np.array_equal((code >> 15) & 1, ((s < 0) ^ (b >= N2)).astype(np.uint32))
    tail_cap = L // 64 * 18
    assert cs == dim or cs == cs_fixed
    for c, c0 in enumerate(range(0, dim, cs)):
        rows = np.arange(c0, min(dim, c0 + cs))
        tp = code[rows] >> 16
        first = {}
        for i in rows:
            first.setdefault(slot[i], i)
        is_first = np.array([first[slot[i]] == i for i in rows])
        assert np.array_equal(tp == 0xFFFF, is_first)
        later = rows[~is_first]
        order = later[np.lexsort((later, slot[later]))]
        assert np.array_equal(code[order] >> 16, np.arange(len(later)))  # tail order (slot, row)
        assert len(later) <= tail_cap
        ng = int(ngroups[c])
        gs = groups[c * (cs // 2):c * (cs // 2) + ng]
        uniq, cnt = np.unique(slot[later], return_counts=True)
        assert ng == len(uniq)
        assert np.array_equal(gs[:, 0] & 0x3FFF, idx(uniq))
        assert np.array_equal(gs[:, 1], cnt)
        assert np.array_equal(gs[:, 0] >> 16, np.concatenate([[0], np.cumsum(cnt)[:-1]]))


def test_split_abi_arguments():
    """Unsupported lengths and missing plans are rejected, not run."""
    assert query("ids_tensorsketch_split_ok", 3, 4096) == 1
    assert query("ids_tensorsketch_split_ok", 3, 2048) == 0
    assert query("ids_tensorsketch_split_ok", 9, 4096) == 0
    n = 1
    fac = torch.zeros((1, 100), dtype=torch.float64, device="cuda")
    y = torch.empty((1, 4096), dtype=torch.float64, device="cuda")
    ptrs = (ctypes.c_void_p * n)(fac.data_ptr())
    dims = (ctypes.c_int64 * n)(100)
    lds = (ctypes.c_int64 * n)(100)
    plans = (ctypes.c_void_p * n)(None)
    with pytest.raises(ValueError):
        call("ids_tensorsketch_split_f64", n, ctypes.addressof(ptrs), ctypes.addressof(dims),
             ctypes.addressof(lds), 1, ctypes.addressof(plans), 4096, None, y.data_ptr(), None, None)


def test_split_without_norms_and_single_term():
    """colnorm2 = NULL (no norm epilogue) gives the same sketch; one term
    column runs on one cluster."""
    rng = np.random.default_rng(17)
    dims, L = [3000, 2500], 16384
    for r in (1, 37):
        fac = _factors(rng, dims, r)
        w = torch.from_numpy(rng.random(r) + 0.5).cuda()
        op = ids.TensorSketchOp(dims, L, seed=2)
        y_n, nrm = op.apply_device(fac, w, norms=True)
        y = op.apply_device(fac, w)
        assert torch.equal(y, y_n)
        assert float(((nrm - (y * y).sum(dim=1)).abs() / nrm).max()) <= 1e-13
        want = oracle.OracleTensorSketch(dims, L, seed=2).apply([f.cpu().numpy() for f in fac],
                                                               w.cpu().numpy())
        assert relerr_fro(y.t().cpu().numpy(), want) <= 1e-12

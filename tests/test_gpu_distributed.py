"""The column-distributed CPQR kernels (csrc/cpqr_dist.cu) on
the GPU: one shard (world 1) and several shards driven in one process with
the real step driver (the collectives replaced by local copies), against
LAPACK's pivots and the reference's coefficients (CPU oracle)."""

import numpy as np
import pytest

import oracle

from conftest import relerr_fro

pytestmark = pytest.mark.gpu

ids = pytest.importorskip("paper_1901_10559_b200")
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1901_10559_b200.distributed import (  # noqa: E402
    DeviceBackend,
    DeviceCpqrShard,
    assemble_pivoted,
    cpqr_columns_sharded,
    dcpqr_steps,
)


def _near_dup(rng, m, n, base, pert):
    b = rng.standard_normal((m, base))
    idx = rng.integers(0, base, size=n)
    idx[:base] = np.arange(base)
    return b[:, idx] + pert * rng.standard_normal((m, n))


def _run_local_shards(y, k, bounds):
    shards = [DeviceCpqrShard(torch.from_numpy(np.ascontiguousarray(y[:, a:b].T)).cuda(), a, k)
              for a, b in zip(bounds[:-1], bounds[1:])]

    def gather(cands):
        return torch.stack(cands).cpu().numpy()

    def broadcast(a_list, cs):
        src = next(i for i, sh in enumerate(shards) if sh.owns(cs))
        for i, a in enumerate(a_list):
            if i != src:
                a.copy_(a_list[src])

    dcpqr_steps(shards, k, gather, broadcast)
    parts = [sh.results() for sh in shards]
    pos = np.concatenate([p[0].cpu().numpy() for p in parts])
    r = np.concatenate([p[1].cpu().numpy() for p in parts], axis=1)
    return assemble_pivoted(pos, r, parts[0][2].cpu().numpy(), k, 1e-12)


@pytest.mark.parametrize("m,n,k,base,pert", [(4096, 1000, 10, 10, 1e-3), (100, 2000, 20, 20, 1e-2),
                                             (16384, 300, 20, 20, 1e-4), (40, 37, 5, 9, 1e-2)])
def test_single_shard_matches_oracle(m, n, k, base, pert):
    y = _near_dup(np.random.default_rng(m + n), m, n, base, pert)
    d = cpqr_columns_sharded(torch.from_numpy(np.ascontiguousarray(y.T)).cuda(), 0, n, k)
    want = oracle.matrix_id(y, k)
    assert np.array_equal(d.cols, want.cols)
    assert relerr_fro(d.coeffs, want.coeffs) <= 1e-10
    assert d.numerical_rank == want.numerical_rank


@pytest.mark.parametrize("bounds", [[0, 300, 600, 1000], [0, 1, 500, 999, 1000], [0, 1000]])
def test_several_shards_match_oracle(bounds):
    y = _near_dup(np.random.default_rng(3), 4096, 1000, 10, 1e-3)
    k = 10
    perm, rtop, nr = _run_local_shards(y, k, bounds)
    want = oracle.cpqr(y, k)
    assert np.array_equal(perm[:k], want.perm[:k])
    mine = np.abs(rtop)[:, np.argsort(perm)]
    ref = np.abs(want.r)[:, np.argsort(want.perm)]
    assert relerr_fro(mine, ref) <= 1e-10
    assert nr == want.numerical_rank
    d = DeviceBackend().coeffs_from_factors(rtop, perm, k, 1000, 1e-12, nr)
    w = oracle.matrix_id(y, k)
    assert np.array_equal(d.cols, w.cols)
    assert relerr_fro(d.coeffs, w.coeffs) <= 1e-10


def test_zero_and_deficient_sketches():
    y = np.zeros((64, 30))
    d = cpqr_columns_sharded(torch.zeros((30, 64), dtype=torch.float64, device="cuda"), 0, 30, 4)
    assert d.numerical_rank == 0 and d.rank_deficient
    assert np.all(np.isfinite(d.coeffs))
    want = oracle.matrix_id(y, 4)
    assert np.array_equal(d.cols, want.cols)
    y = _near_dup(np.random.default_rng(5), 64, 40, 5, 0.0)  # exact rank 5 < k
    perm, rtop, nr = _run_local_shards(y, 12, [0, 13, 40])
    w = oracle.matrix_id(y, 12)
    assert nr == w.numerical_rank
    assert np.array_equal(perm[:nr], w.cols[:nr])


def _run_local_shards_device(y, k, bounds):
    """The device-driven loop of cpqr_columns_sharded with the collectives
    replaced by local ops: cat of the candidates, a plain sum of the pivot
    columns (non-owners contribute -0.0)."""
    shards = [DeviceCpqrShard(torch.from_numpy(np.ascontiguousarray(y[:, a:b].T)).cuda(), a, k)
              for a, b in zip(bounds[:-1], bounds[1:])]
    for kk in range(k):
        c = torch.cat([sh.cand.reshape(1, 4) for sh in shards])
        pivs = [sh.select(c, kk) for sh in shards]
        a_list = [sh.pivot_dev(kk, p) for sh, p in zip(shards, pivs)]
        tot = a_list[0].clone()
        for a in a_list[1:]:
            tot += a
        for sh, p in zip(shards, pivs):
            sh.step_dev(kk, p, tot)
    parts = [sh.results() for sh in shards]
    pos = np.concatenate([p[0].cpu().numpy() for p in parts])
    r = np.concatenate([p[1].cpu().numpy() for p in parts], axis=1)
    return assemble_pivoted(pos, r, parts[0][2].cpu().numpy(), k, 1e-12)


@pytest.mark.parametrize("bounds", [[0, 300, 600, 1000], [0, 1, 500, 999, 1000], [0, 1000]])
def test_device_driven_steps_bit_identical(bounds):
    """Pivot picked on the device + summed pivot column == the host-driven
    steps (host pick + broadcast), bit for bit; pivots equal LAPACK's."""
    y = _near_dup(np.random.default_rng(3), 4096, 1000, 10, 1e-3)
    y[:, 17] = 0.0  # an exactly zero column (its +-0 entries must survive the sum)
    k = 10
    p1, r1, n1 = _run_local_shards(y, k, bounds)
    p2, r2, n2 = _run_local_shards_device(y, k, bounds)
    assert np.array_equal(p1, p2) and n1 == n2
    assert np.array_equal(r1, r2)
    assert np.array_equal(p2[:k], oracle.cpqr(y, k).perm[:k])


def test_device_driven_zero_sketch():
    y = np.zeros((64, 30))
    p1, r1, n1 = _run_local_shards(y, 4, [0, 10, 30])
    p2, r2, n2 = _run_local_shards_device(y, 4, [0, 10, 30])
    assert np.array_equal(p1, p2) and n1 == n2 == 0
    assert np.array_equal(np.signbit(r1), np.signbit(r2)) and np.array_equal(r1, r2)


def _run_local_shards_fused(y, k, bounds):
    """As _run_local_shards_device, with select + pivot in one launch
    (ids_dcpqr_select_pivot_f64), as distributed.py drives it."""
    shards = [DeviceCpqrShard(torch.from_numpy(np.ascontiguousarray(y[:, a:b].T)).cuda(), a, k)
              for a, b in zip(bounds[:-1], bounds[1:])]
    for kk in range(k):
        c = torch.cat([sh.cand.reshape(1, 4) for sh in shards])
        outs = [sh.select_pivot(c, kk) for sh in shards]
        tot = outs[0][1].clone()
        for _, a in outs[1:]:
            tot += a
        for sh, (p, _) in zip(shards, outs):
            sh.step_dev(kk, p, tot)
    parts = [sh.results() for sh in shards]
    pos = np.concatenate([p[0].cpu().numpy() for p in parts])
    r = np.concatenate([p[1].cpu().numpy() for p in parts], axis=1)
    return assemble_pivoted(pos, r, parts[0][2].cpu().numpy(), k, 1e-12)


@pytest.mark.parametrize("shape,bounds", [((4096, 1000), [0, 300, 600, 1000]),
                                          ((4096, 1000), [0, 1, 500, 999, 1000]),
                                          ((16384, 250), [0, 250]), ((700, 90), [0, 45, 90])])
def test_fused_steps_bit_identical(shape, bounds):
    """The fused select+pivot kernel reproduces the separate select and
    pivot kernels bit for bit."""
    m, n = shape
    y = _near_dup(np.random.default_rng(m + n), m, n, 10, 1e-3)
    y[:, 17] = 0.0
    k = 10
    p1, r1, n1 = _run_local_shards_device(y, k, bounds)
    p2, r2, n2 = _run_local_shards_fused(y, k, bounds)
    assert np.array_equal(p1, p2) and n1 == n2
    assert np.array_equal(r1, r2)
    assert np.array_equal(p2[:k], oracle.cpqr(y, k).perm[:k])

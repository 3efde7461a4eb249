"""The multi-GPU partitioning and collectives (paper_1901_10559_b200.distributed)
exercised on CPU: world_size 2 over gloo, with the CPU oracle as the
per-shard arithmetic backend.  The GPU backend runs the same host logic."""

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1901_10559_b200.distributed import (
    countsketch_id_sharded,
    cpqr_columns_sharded,
    row_block,
    tensorsketch_id_sharded,
)


class OracleBackend:
    """Per-shard arithmetic on the CPU oracle (test infrastructure)."""

    def matrix_sketch(self, a_local, row0, in_dim, sketch_dim, seed, surjective):
        op = oracle.OracleCountSketch(in_dim, sketch_dim, seed, surjective)
        rows = a_local.shape[0]
        y = oracle.cs_apply(op.bucket[row0:row0 + rows], op.sign[row0:row0 + rows],
                            sketch_dim, a_local)
        flag = torch.tensor([0 if np.isfinite(y).all() else 1], dtype=torch.int32)
        return torch.from_numpy(np.ascontiguousarray(y.T)), flag, a_local

    def confirm_nonfinite(self, operand):
        return torch.tensor([0 if np.isfinite(operand).all() else 1], dtype=torch.int32)

    def tensor_sketch(self, factors, weights, mode_dims, sketch_dim, seed):
        y = oracle.OracleTensorSketch(mode_dims, sketch_dim, seed).apply(factors, weights)
        return torch.from_numpy(np.ascontiguousarray(y.T))

    def matrix_id(self, y, rows, cols, rank, rank_tol, method):
        return oracle.matrix_id(y.numpy().T, rank, rank_tol)

    def cpqr_shard(self, y_local, col0, k):
        return oracle.OracleCpqrShard(y_local, col0, k)

    def coeffs_from_factors(self, rtop, perm, k, ncols, rank_tol, numerical_rank):
        coeffs, deficient = oracle.coeffs_from_pivoted(rtop, perm, k, numerical_rank, rank_tol)
        return SimpleNamespace(cols=perm[:k].astype(np.int32), coeffs=coeffs,
                               numerical_rank=numerical_rank, rank_deficient=deficient)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _matrix_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        a = rng.standard_normal((2003, 8)) @ rng.standard_normal((8, 60))
        a += 1e-3 * rng.standard_normal(a.shape)
        r0, r1 = row_block(a.shape[0], world, rank)
        d = countsketch_id_sharded(a[r0:r1], r0, a.shape[0], 8, 30, seed=5,
                                   backend=OracleBackend())
        bad = a[r0:r1].copy()
        if rank == 1:
            bad[3, 2] = np.nan
        try:
            countsketch_id_sharded(bad, r0, a.shape[0], 8, 30, seed=5, backend=OracleBackend())
            raised = False
        except ValueError:
            raised = True
        out[rank] = (d.cols.tolist(), d.coeffs.tolist(), raised)
    finally:
        dist.destroy_process_group()


def _tensor_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(1)
        R = 41
        fac = [rng.standard_normal((d, R)) for d in (9, 8, 7)]
        w = rng.random(R) + 0.5
        c0, c1 = row_block(R, world, rank)
        x_local = SimpleNamespace(factors=[f[:, c0:c1] for f in fac], weights=w[c0:c1],
                                  mode_dims=(9, 8, 7))
        res = {}
        for mode in ("columns", "gather"):
            d, nw = tensorsketch_id_sharded(x_local, c0, R, w, 6, 64, seed=3,
                                            backend=OracleBackend(), cpqr=mode)
            res[mode] = (d.cols.tolist(), d.coeffs.tolist(), nw.tolist())
        out[rank] = res
    finally:
        dist.destroy_process_group()


def _run(worker, world=2):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(worker, args=(world, _free_port(), out), nprocs=world, join=True)
    return dict(out)


def test_row_block_partition():
    for n in (1, 7, 1000, 10**6 + 3):
        for world in (1, 2, 3, 8):
            blocks = [row_block(n, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))


def test_countsketch_id_row_sharded_gloo():
    out = _run(_matrix_worker)
    rng = np.random.default_rng(0)
    a = rng.standard_normal((2003, 8)) @ rng.standard_normal((8, 60))
    a += 1e-3 * rng.standard_normal(a.shape)
    want = oracle.countsketch_id(a, 8, 30, seed=5)
    for rank in (0, 1):
        cols, coeffs, raised = out[rank]
        assert cols == want.cols.tolist()
        c = np.array(coeffs)
        assert np.linalg.norm(c - want.coeffs) <= 1e-10 * np.linalg.norm(want.coeffs)
        assert raised  # a NaN on one shard raises on every rank
    assert out[0][1] == out[1][1]  # identical on all ranks


def test_tensorsketch_id_term_sharded_gloo():
    out = _run(_tensor_worker)
    rng = np.random.default_rng(1)
    R = 41
    fac = [rng.standard_normal((d, R)) for d in (9, 8, 7)]
    w = rng.random(R) + 0.5
    want, nw = oracle.tensorsketch_id(w, fac, 6, 64, seed=3)
    for rank in (0, 1):
        cols, coeffs, new_w = out[rank]["gather"]
        assert cols == want.cols.tolist()
        # the term-sharded sketch is bit-identical to the unsharded one
        assert np.array_equal(np.array(coeffs), want.coeffs)
        assert np.array_equal(np.array(new_w), nw)
        # column-distributed CPQR: same pivots, P within the fp64 tolerance
        cols, coeffs, new_w = out[rank]["columns"]
        assert cols == want.cols.tolist()
        assert np.linalg.norm(np.array(coeffs) - want.coeffs) <= 1e-10 * np.linalg.norm(want.coeffs)
        assert np.abs(np.array(new_w) - nw).max() <= 1e-10 * np.abs(nw).max()
    assert out[0]["columns"] == out[1]["columns"]  # identical on all ranks


def _near_dup(rng, m, n, base, pert):
    b = rng.standard_normal((m, base))
    idx = rng.integers(0, base, size=n)
    idx[:base] = np.arange(base)
    return b[:, idx] + pert * rng.standard_normal((m, n))


def _dcpqr_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        for case, (m, n, k, base, pert) in enumerate([(300, 101, 8, 8, 1e-3), (64, 40, 12, 5, 0.0),
                                                     (50, 7, 3, 7, 1e-2)]):
            y = _near_dup(np.random.default_rng(case), m, n, base, pert)
            c0, c1 = row_block(n, world, rank)
            y_local = torch.from_numpy(np.ascontiguousarray(y[:, c0:c1].T))
            d = cpqr_columns_sharded(y_local, c0, n, k, backend=OracleBackend())
            res.append((d.cols.tolist(), d.coeffs.tolist(), d.numerical_rank, d.rank_deficient))
        out[rank] = res
    finally:
        dist.destroy_process_group()


def test_column_distributed_cpqr_gloo():
    """three ranks with uneven column blocks (one rank-deficient
    case) agree with LAPACK's pivots and the reference's coefficients."""
    out = _run(_dcpqr_worker, world=3)
    for case, (m, n, k, base, pert) in enumerate([(300, 101, 8, 8, 1e-3), (64, 40, 12, 5, 0.0),
                                                 (50, 7, 3, 7, 1e-2)]):
        y = _near_dup(np.random.default_rng(case), m, n, base, pert)
        want = oracle.matrix_id(y, k)
        for rank in range(3):
            cols, coeffs, nr, deficient = out[rank][case]
            assert nr == want.numerical_rank and deficient == want.rank_deficient
            nr_ = want.numerical_rank
            assert cols[:nr_] == want.cols[:nr_].tolist(), case
            if not deficient:
                c = np.array(coeffs)
                assert np.linalg.norm(c - want.coeffs) <= 1e-9 * np.linalg.norm(want.coeffs)
        assert out[0][case] == out[1][case] == out[2][case]


def test_column_distributed_cpqr_local_shards():
    """The step driver with several shards in one process (no collectives)."""
    from paper_1901_10559_b200.distributed import assemble_pivoted, dcpqr_steps

    rng = np.random.default_rng(7)
    y = _near_dup(rng, 120, 57, 6, 1e-4)
    k = 6
    bounds = [0, 10, 11, 40, 57]  # includes a one-column shard
    shards = [oracle.OracleCpqrShard(np.ascontiguousarray(y[:, a:b].T), a, k)
              for a, b in zip(bounds[:-1], bounds[1:])]

    def gather(cands):
        return torch.stack(cands).numpy()

    def broadcast(a_list, cs):
        src = next(i for i, sh in enumerate(shards) if sh.owns(cs))
        for i, a in enumerate(a_list):
            if i != src:
                a.copy_(a_list[src])

    dcpqr_steps(shards, k, gather, broadcast)
    parts = [sh.results() for sh in shards]
    pos = np.concatenate([p[0].numpy() for p in parts])
    r = np.concatenate([p[1].numpy() for p in parts], axis=1)
    perm, rtop, nr = assemble_pivoted(pos, r, parts[0][2].numpy(), k, 1e-12)
    want = oracle.cpqr(y, k)
    assert np.array_equal(perm[:k], want.perm[:k])
    mine = np.abs(rtop)[:, np.argsort(perm)]
    ref = np.abs(want.r)[:, np.argsort(want.perm)]
    assert np.linalg.norm(mine - ref) <= 1e-10 * np.linalg.norm(ref)
    assert nr == want.numerical_rank


if __name__ == "__main__":  # pragma: no cover
    pytest.main([__file__, "-q"])


def _entropy_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1901_10559_b200.distributed import _agreed_entropy

        sub = dist.new_group([1, 0][:world])  # a subgroup: src must be a GLOBAL rank
        vals = [_agreed_entropy(None), _agreed_entropy(sub)]
        # seed=None: every rank draws the same hash (fresh entropy agreed on)
        rng = np.random.default_rng(3)
        a = rng.standard_normal((500, 6)) @ rng.standard_normal((6, 40))
        r0, r1 = row_block(500, world, rank)
        d = countsketch_id_sharded(a[r0:r1], r0, 500, 6, 20, seed=None, backend=OracleBackend())
        try:
            cpqr_columns_sharded(torch.zeros((3, 20), dtype=torch.float64), 5, 40, 2,
                                 backend=OracleBackend())
            bad_split = False
        except ValueError:
            bad_split = True
        out[rank] = (vals, d.cols.tolist(), bad_split)
    finally:
        dist.destroy_process_group()


def test_seed_none_agreement_and_split_check_gloo():
    out = _run(_entropy_worker)
    assert out[0][0] == out[1][0]  # same entropy on every rank, default and subgroup
    assert out[0][1] == out[1][1]  # same hash -> same decomposition
    assert out[0][2] and out[1][2]  # a column block off the row_block split is rejected

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
        d, nw = tensorsketch_id_sharded(x_local, c0, R, w, 6, 64, seed=3,
                                        backend=OracleBackend())
        out[rank] = (d.cols.tolist(), d.coeffs.tolist(), nw.tolist())
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
        cols, coeffs, new_w = out[rank]
        assert cols == want.cols.tolist()
        # the term-sharded sketch is bit-identical to the unsharded one
        assert np.array_equal(np.array(coeffs), want.coeffs)
        assert np.array_equal(np.array(new_w), nw)


if __name__ == "__main__":  # pragma: no cover
    pytest.main([__file__, "-q"])

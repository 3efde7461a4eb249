"""The multi-GPU code paths with their real device kernels: two ranks over
gloo, both on cuda:0 (gloo's collectives are host-staged, so no kernel of one
rank waits on the other's).  Row-sharded countsketch_id (single call and the
pipelined trials), the NaN agreement across ranks, and the term-sharded
tensor ID with the column-distributed CPQR, against one-process results."""

import os
import socket

import numpy as np
import pytest

import oracle

from conftest import relerr_fro

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix():
    rng = np.random.default_rng(41)
    a = rng.standard_normal((6001, 12)) @ rng.standard_normal((12, 90))
    return a + 1e-4 * rng.standard_normal(a.shape)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1901_10559_b200 as ids
        from paper_1901_10559_b200.distributed import (
            countsketch_id_sharded, countsketch_id_sharded_trials, row_block,
            tensorsketch_id_sharded)

        a = _matrix()
        r0, r1 = row_block(a.shape[0], world, rank)
        local = torch.from_numpy(np.ascontiguousarray(a[r0:r1])).cuda()
        d = countsketch_id_sharded(local, r0, a.shape[0], 12, 40, seed=3)
        trials = countsketch_id_sharded_trials(local, r0, a.shape[0], 12, 40, seeds=[3, 4, 5])
        bad = a[r0:r1].copy()
        if rank == 1:
            bad[2, 5] = np.inf
        try:
            countsketch_id_sharded_trials(torch.from_numpy(bad).cuda(), r0, a.shape[0], 12, 40,
                                          seeds=[6, 7])
            raised = False
        except ValueError:
            raised = True
        rng = np.random.default_rng(42)
        R = 37
        fac = [rng.standard_normal((d_, R)) for d_ in (11, 9, 8)]
        w = rng.random(R) + 0.5
        x = ids.CpTensor(w, fac)
        c0, c1 = row_block(R, world, rank)
        from types import SimpleNamespace
        xl = SimpleNamespace(factors=[f[:, c0:c1] for f in x.factors], weights=x.weights[c0:c1],
                             mode_dims=x.mode_dims)
        td, nw = tensorsketch_id_sharded(xl, c0, R, x.weights, 5, 64, seed=8)
        # trial-sharded hash draws: every rank gets every trial's hash, drawn by
        # one owner rank and broadcast; compare with local draws bit for bit
        from paper_1901_10559_b200.distributed import trial_sharded_operators
        hashes_ok = []
        for s_, op in zip([9, 10, 11, 12, 13],
                          trial_sharded_operators(a.shape[0], 40, [9, 10, 11, 12, 13], True)):
            local_op = ids.CountSketchOp(a.shape[0], 40, seed=s_, surjective=True)
            hashes_ok.append(bool(np.array_equal(op.bucket, local_op.bucket)
                                  and np.array_equal(op.sign, local_op.sign)
                                  and op.draws == local_op.draws))
        out[rank] = {
            "hashes_ok": hashes_ok,
            "cols": d.cols.tolist(), "coeffs": d.coeffs.tolist(),
            "trials": [(t.cols.tolist(), t.coeffs.tolist()) for t in trials],
            "raised": raised,
            "tcols": td.cols.tolist(), "tcoeffs": td.coeffs.tolist(), "nw": nw.tolist(),
        }
    finally:
        dist.destroy_process_group()


def test_row_and_term_sharding_on_device_kernels():
    import paper_1901_10559_b200 as ids

    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _port(), out), nprocs=2, join=True)
    out = dict(out)
    a = _matrix()
    want = ids.countsketch_id(a, 12, 40, seed=3)
    ref = oracle.countsketch_id(a, 12, 40, seed=3)
    assert np.array_equal(want.cols, ref.cols)
    for rank in (0, 1):
        o = out[rank]
        assert o["cols"] == want.cols.tolist()
        # shard-boundary rounding (the all-reduce adds two partial sums)
        assert relerr_fro(np.array(o["coeffs"]), want.coeffs) <= 1e-10
        for (cols, coeffs), seed in zip(o["trials"], (3, 4, 5)):
            single = ids.countsketch_id(a, 12, 40, seed=seed)
            assert cols == single.cols.tolist()
            assert relerr_fro(np.array(coeffs), single.coeffs) <= 1e-10
        assert o["raised"]  # an Inf on one rank raises on every rank
    assert out[0]["coeffs"] == out[1]["coeffs"]
    assert out[0]["hashes_ok"] == [True] * 5 and out[1]["hashes_ok"] == [True] * 5
    rng = np.random.default_rng(42)
    R = 37
    fac = [rng.standard_normal((d_, R)) for d_ in (11, 9, 8)]
    x = ids.CpTensor(rng.random(R) + 0.5, fac)
    tw = ids.tensorsketch_id(x, 5, 64, seed=8)
    for rank in (0, 1):
        o = out[rank]
        assert o["tcols"] == tw.cols.tolist()
        assert relerr_fro(np.array(o["tcoeffs"]), tw.coeffs) <= 1e-10
        assert relerr_fro(np.array(o["nw"]), tw.new_weights) <= 1e-10
    assert out[0]["tcoeffs"] == out[1]["tcoeffs"]

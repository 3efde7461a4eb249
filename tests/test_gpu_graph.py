"""Seeds read from device memory (ids_countsketch_hash_dev) and the
CUDA-graph tensor ID (TensorIdGraph): bit-identical to the eager path."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ids = pytest.importorskip("paper_1901_10559_b200")
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_1901_10559_b200 import generators as G  # noqa: E402


@pytest.mark.parametrize("I,L,surj", [(100_000, 200, True), (4097, 64, False), (1000, 4096, False)])
def test_hash_seed_from_device_memory(I, L, surj):
    st = ids.TensorSketchOp.mode_seed_states(3, 77)
    for n in range(3):
        dev = torch.from_numpy(st[n].copy()).cuda()
        a = ids.CountSketchOp(I, L, seed=np.random.SeedSequence([77, n]), surjective=surj)
        b = ids.CountSketchOp(I, L, surjective=surj, _seed_dev=dev)
        assert np.array_equal(a.bucket, b.bucket) and np.array_equal(a.sign, b.sign)
        assert a.draws == b.draws


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_tensor_id_graph_matches_eager(name):
    cfg = G.CONFIGS[name]
    w, facs = G.cp_config(name)
    x = ids.CpTensor(w.cpu().numpy(), [f.cpu().numpy() for f in facs])
    g = ids.TensorIdGraph(facs, w, cfg["k"], cfg["L"], host_weights=x.weights)
    for seed in (3, 11, 3):
        d, nw = g(seed)
        want = ids.tensorsketch_id(x, cfg["k"], cfg["L"], seed=seed)
        assert np.array_equal(d.cols, want.cols)
        assert np.array_equal(d.coeffs, want.coeffs)
        assert np.array_equal(nw, want.new_weights)
        assert d.numerical_rank == want.numerical_rank


def test_tensor_id_graph_trials():
    cfg = G.CONFIGS["C4"]
    w, facs = G.cp_config("C4")
    x = ids.CpTensor(w.cpu().numpy(), [f.cpu().numpy() for f in facs])
    g = ids.TensorIdGraph(facs, w, cfg["k"], cfg["L"], host_weights=x.weights)
    out = g.trials([5, 6, 7, 5])
    for (d, nw), s in zip(out, [5, 6, 7, 5]):
        want = ids.tensorsketch_id(x, cfg["k"], cfg["L"], seed=s)
        assert np.array_equal(d.cols, want.cols) and np.array_equal(d.coeffs, want.coeffs)
        assert np.array_equal(nw, want.new_weights)


@pytest.mark.parametrize("seeds", [[1, 2, 3], [9, 8, 7, 6, 5, 4, 3], [4, 4, 4, 4]])
def test_tensor_id_graph_pipelined_trials_equal_sequential(seeds):
    # trials on two twin graphs (next trial's draws beside this trial's
    # compute) against replays of one graph, and two trials (below the
    # pipelining threshold) against both
    cfg = G.CONFIGS["C4"]
    w, facs = G.cp_config("C4")
    g = ids.TensorIdGraph(facs, w, cfg["k"], cfg["L"])
    seq = ids.TensorIdGraph(facs, w, cfg["k"], cfg["L"], pipeline_trials=False)
    for rep in range(2):  # the twins are reused by a second call
        for (da, na), (db, nb) in zip(g.trials(seeds), seq.trials(seeds)):
            assert np.array_equal(da.cols, db.cols) and np.array_equal(da.coeffs, db.coeffs)
            assert np.array_equal(na, nb) and da.numerical_rank == db.numerical_rank
    assert g._twin_graphs is not None and seq._twin_graphs is None
    for (da, na), (db, nb) in zip(g.trials(seeds[:2]), seq.trials(seeds[:2])):
        assert np.array_equal(da.cols, db.cols) and np.array_equal(da.coeffs, db.coeffs)


def test_device_cp_tensor_matches_host():
    """CpTensor over CUDA factors (normalized on the device, kept in HBM):
    tensorsketch_id gives the host path's results (bit-identical for unit
    columns, 1e-13 when the device rescales), the reduced tensor stays on the
    device, and the sign fix / zero columns follow cp_tensor.py:52-95."""
    rng = np.random.default_rng(8)
    w, facs = G.cp_config("C4")
    xh = ids.CpTensor(w.cpu().numpy(), [f.cpu().numpy() for f in facs])
    xd = ids.CpTensor(w.cpu().numpy(), facs)
    assert all(f.is_cuda and f.t().is_contiguous() for f in xd.factors)
    a = ids.tensorsketch_id(xh, 10, 4096, seed=2)
    b = ids.tensorsketch_id(xd, 10, 4096, seed=2)
    assert np.array_equal(a.cols, b.cols) and np.array_equal(a.coeffs, b.coeffs)
    assert np.array_equal(a.new_weights, b.new_weights)
    assert b.reduced.factors[0].is_cuda
    assert ids.cp_diff_norm(xd, b.reduced) == pytest.approx(ids.cp_diff_norm(xh, a.reduced),
                                                            rel=1e-12)
    # unnormalized columns, a negative weight, a zero column
    fh = [rng.standard_normal((40, 6)) * 3.0 for _ in range(3)]
    fh[1][:, 4] = 0.0
    wh = np.array([1.0, -2.0, 0.5, 1.5, 1.0, 0.7])
    xh = ids.CpTensor(wh, fh)
    xd = ids.CpTensor(wh, [torch.from_numpy(f).cuda() for f in fh])
    assert np.allclose(xd.weights, xh.weights, rtol=1e-14) and (xd.weights >= 0).all()
    assert np.array_equal(xd.zero_columns, xh.zero_columns)
    for u, v in zip(xd.factors, xh.factors):
        assert np.allclose(u.cpu().numpy(), v, rtol=0, atol=1e-15)
    ra, rb = ids.tensorsketch_id(xh, 3, 30, seed=1), ids.tensorsketch_id(xd, 3, 30, seed=1)
    assert np.array_equal(ra.cols, rb.cols)
    assert np.allclose(ra.coeffs, rb.coeffs, rtol=1e-12, atol=1e-13)


def test_tensor_id_graph_rejects_host_inputs():
    with pytest.raises(ValueError):
        ids.TensorIdGraph([np.ones((5, 3))] * 2, np.ones(3), 2, 8)


def _eager(x, k, L, seed):
    from paper_1901_10559_b200 import cp_tensor

    cp_tensor.HOST_GRAPHS = False
    try:
        return ids.tensorsketch_id(x, k, L, seed=seed)
    finally:
        cp_tensor.HOST_GRAPHS = True


def _same(a, b):
    assert np.array_equal(a.cols, b.cols)
    assert np.array_equal(a.coeffs, b.coeffs)
    assert np.array_equal(a.new_weights, b.new_weights)
    assert a.numerical_rank == b.numerical_rank and a.rank_deficient == b.rank_deficient
    assert all(np.array_equal(p, q) for p, q in zip(a.reduced.factors, b.reduced.factors))
    assert np.array_equal(a.reduced.weights, b.reduced.weights)


@pytest.mark.parametrize("pinned", [False, True])
def test_host_tensor_repeat_calls_replay_graph(pinned):
    """tensorsketch_id on host factors: the second call of a shape captures
    a graph over device copies of the factors, later calls refill them and
    replay; every result equals the eager path's, also when shapes alternate
    and when the factor values change between calls."""
    from paper_1901_10559_b200 import cp_tensor

    rng = np.random.default_rng(4)

    def tensor(dims, R, scale=1.0):
        fs = []
        for d in dims:
            f = torch.from_numpy(rng.standard_normal((R, d)) * scale)
            f = f / f.norm(dim=1, keepdim=True)
            fs.append((f.pin_memory() if pinned else f).numpy().T)
        return ids.CpTensor(rng.random(R) + 0.1, fs)

    xa, xb = tensor((300, 200, 90), 400), tensor((5000, 64), 300)
    for x, k, L, seed in [(xa, 10, 4096, 1), (xa, 10, 4096, 2), (xa, 10, 4096, 3),
                          (xb, 7, 1024, 4), (xb, 7, 1024, 5), (xa, 10, 4096, 6),
                          (xa, 10, 4096, 7)]:
        _same(ids.tensorsketch_id(x, k, L, seed=seed), _eager(x, k, L, seed))
    assert cp_tensor._host_graph["graph"] is not None
    xc = tensor((300, 200, 90), 400, scale=3.0)  # same shape, new values
    _same(ids.tensorsketch_id(xc, 10, 4096, seed=8), _eager(xc, 10, 4096, 8))


def test_split_graph_matches_single_graph():
    """TensorIdGraph(split=True) (draw and compute graphs) gives the single
    graph's results, through __call__ and trials()."""
    w, facs = G.cp_config("C4")
    cfg = G.CONFIGS["C4"]
    a = ids.TensorIdGraph(facs, w, cfg["k"], cfg["L"])
    b = ids.TensorIdGraph(facs, w, cfg["k"], cfg["L"], split=True)
    for seed in (5, 6):
        (da, na), (db, nb) = a(seed), b(seed)
        assert np.array_equal(da.cols, db.cols) and np.array_equal(da.coeffs, db.coeffs)
        assert np.array_equal(na, nb)
    for (da, na), (db, nb) in zip(a.trials([1, 2, 3]), b.trials([1, 2, 3])):
        assert np.array_equal(da.cols, db.cols) and np.array_equal(da.coeffs, db.coeffs)
        assert np.array_equal(na, nb)


def test_host_tensor_graph_concurrent_threads():
    """Calls from several threads: one owns the cached graph at a time, the
    others run eagerly; every result equals the eager path's."""
    import threading

    rng = np.random.default_rng(9)
    facs = []
    for d in (300, 200, 90):
        f = rng.standard_normal((d, 400))
        facs.append(np.asfortranarray(f / np.linalg.norm(f, axis=0)))
    x = ids.CpTensor(rng.random(400) + 0.1, facs)
    want = {s: _eager(x, 10, 4096, s) for s in range(8)}
    got, errs = {}, []

    def work(seeds):
        try:
            for s in seeds:
                got[s] = ids.tensorsketch_id(x, 10, 4096, seed=s)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=work, args=([s, s + 4],)) for s in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs
    for s in range(8):
        _same(got[s], want[s])

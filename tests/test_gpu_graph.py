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

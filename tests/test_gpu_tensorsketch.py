"""TensorSketch + tensor ID parity on the GPU against the golden fixtures
(pocketfft / LAPACK via the real reference) and the CPU oracle."""

import numpy as np
import pytest
import scipy.sparse as sp

import oracle

from conftest import dense_countsketch, khatri_rao, relerr_fro

pytestmark = pytest.mark.gpu

ids = pytest.importorskip("paper_1901_10559_b200")
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

TOL = 1e-10


def test_tensorsketch_golden(golden):
    data, man = golden
    for case in man["tensorsketch"]:
        n = case["id"]
        factors = [data[f"ts{n}_f{m}"] for m in range(len(case["dims"]))]
        ts = ids.TensorSketchOp(case["dims"], case["out_dim"], seed=case["seed"])
        y = ts.apply(factors, data[f"ts{n}_w"])
        want = data[f"ts{n}_y"]
        assert y.shape == want.shape
        # per-mode CountSketches are bit-exact; only the FFT rounding differs
        assert relerr_fro(y, want) <= 1e-12, (n, relerr_fro(y, want))


def test_per_mode_hashes_bit_exact():
    ts = ids.TensorSketchOp([1000, 1000, 1000], 4096, seed=0)
    ots = oracle.OracleTensorSketch([1000, 1000, 1000], 4096, seed=0)
    for a, b in zip(ts.mode_ops, ots.mode_ops):
        assert np.array_equal(a.bucket, b.bucket) and np.array_equal(a.sign, b.sign)
    assert ts.seed == 0


def test_single_mode_reduces_to_countsketch():
    rng = np.random.default_rng(7)
    a = rng.standard_normal((12, 5))
    lam = rng.random(5) + 0.5
    op = ids.TensorSketchOp([12], 8, seed=8)
    via_fft = op.apply([a], lam)
    direct = op.mode_ops[0].apply(a * lam)
    assert np.abs(via_fft - direct).max() <= 1e-12


@pytest.mark.parametrize("seed", range(100))
def test_composite_hash_identity(seed):
    """reference acceptance criterion 2 (test_acceptance.py:108-131)."""
    rng = np.random.default_rng(1000 + seed)
    n_modes = 2 if seed % 2 == 0 else 3
    dims = [int(rng.integers(2, 7)) for _ in range(n_modes)]
    r = int(rng.integers(1, 6))
    out_dim = int(rng.integers(2, 17))
    factors = [rng.standard_normal((d, r)) for d in dims]
    lam = rng.random(r) + 0.5
    op = ids.TensorSketchOp(dims, out_dim, seed=seed)
    bucket = np.zeros(1, dtype=np.int64)
    sign = np.ones(1)
    for mode in op.mode_ops:
        bucket = (bucket[:, None] + mode.bucket[None, :]).ravel()
        sign = (sign[:, None] * mode.sign[None, :]).ravel()
    dense_t = dense_countsketch(bucket % out_dim, sign, out_dim)
    m = khatri_rao(factors) * lam
    assert relerr_fro(op.apply(factors, lam), dense_t @ m) <= 1e-12


def test_materialize_and_all_ones():
    factors = [np.ones((2, 1))] * 3
    op = ids.TensorSketchOp([2, 2, 2], 5, seed=9)
    out = op.apply(factors, np.array([1.0]))
    oracle_y = op.materialize() @ khatri_rao(factors)
    assert np.abs(out - oracle_y).max() <= 1e-12
    assert out.sum() == pytest.approx(op.composite_sign().sum(), abs=1e-10)


def test_sparse_factors():
    rng = np.random.default_rng(10)
    factors = [sp.random_array((9, 4), density=0.4, rng=rng, format="csc") for _ in range(3)]
    op = ids.TensorSketchOp([9, 9, 9], 6, seed=11)
    want = op.materialize() @ khatri_rao([f.toarray() for f in factors])
    assert np.abs(op.apply(factors) - want).max() <= 1e-11


def test_mismatched_columns():
    op = ids.TensorSketchOp([3, 3], 4, seed=0)
    with pytest.raises(ValueError):
        op.apply([np.ones((3, 2)), np.ones((3, 3))])


@pytest.mark.parametrize("L", [1, 2, 3, 7, 64, 100, 1000, 1452, 2048, 4096, 8192, 16384])
def test_lengths_vs_oracle(L):
    rng = np.random.default_rng(L)
    dims = [50, 40, 30]
    factors = [rng.standard_normal((d, 6)) for d in dims]
    lam = rng.random(6) + 0.5
    op = ids.TensorSketchOp(dims, L, seed=3)
    want = oracle.OracleTensorSketch(dims, L, seed=3).apply(factors, lam)
    assert relerr_fro(op.apply(factors, lam), want) <= 1e-12


def test_tensorsketch_id_golden(golden):
    data, man = golden
    case = man["tensorsketch_id"][0]
    factors = [data[f"tsid_f{m}"] for m in range(len(case["dims"]))]
    x = ids.CpTensor(data["tsid_w"], factors)
    res = ids.tensorsketch_id(x, case["rank"], case["sketch_dim"], seed=case["seed"])
    assert np.array_equal(res.cols, data["tsid_cols"])
    assert relerr_fro(res.coeffs, data["tsid_coeffs"]) <= TOL
    assert relerr_fro(res.new_weights, data["tsid_new_weights"]) <= TOL
    expected = x.weights[res.cols] * res.coeffs.sum(axis=1)
    assert np.array_equal(res.new_weights, expected)
    assert res.method == "tensorsketch"


def _near_dup_cp(rng, dims, R, base, pert):
    bases = rng.integers(0, base, size=R)
    bases[:base] = np.arange(base)
    fac = []
    for d in dims:
        f = rng.standard_normal((d, R))
        f[:, :base] /= np.linalg.norm(f[:, :base], axis=0)
        g = f[:, bases] + pert * rng.standard_normal((d, R))
        g[:, :base] = f[:, :base]
        fac.append(g / np.linalg.norm(g, axis=0))
    return rng.uniform(0.5, 1.0, size=R), fac


def test_config4_full_size_vs_oracle():
    """BASELINE.json configs[3]: N = 3, I = 1000, R = 1000, K = 10, L = 4096."""
    rng = np.random.default_rng(4)
    w, fac = _near_dup_cp(rng, [1000] * 3, 1000, 10, 1e-3)
    x = ids.CpTensor(w, fac)
    for seed in range(3):
        want, nw = oracle.tensorsketch_id(x.weights, x.factors, 10, 4096, seed=seed)
        op = ids.TensorSketchOp(x.mode_dims, 4096, seed=seed)
        y = op.apply(x.factors, x.weights)
        assert relerr_fro(y, want.sketch) <= TOL
        res = ids.tensorsketch_id(x, 10, 4096, seed=seed)
        assert np.array_equal(res.cols, want.cols), seed
        assert relerr_fro(res.coeffs, want.coeffs) <= TOL
        assert relerr_fro(res.new_weights, nw) <= TOL
        err = oracle.cp_diff_norm(x.weights, x.factors, res.reduced.weights, res.reduced.factors)
        ref = oracle.cp_diff_norm(
            x.weights, x.factors, nw, [f[:, want.cols] for f in x.factors])
        assert abs(err - ref) <= 0.01 * ref + 1e-12


def test_exact_rank_recovery_and_keep_all():
    rng = np.random.default_rng(8)
    k, total = 4, 10
    factors = [rng.standard_normal((6, k)) for _ in range(3)]
    weights = np.concatenate([rng.random(k) + 0.5, np.full(total - k, 1e-14)])
    dup = rng.integers(0, k, size=total - k)
    x = ids.CpTensor(weights, [np.hstack([f, f[:, dup]]) for f in factors])
    res = ids.tensorsketch_id(x, k, seed=1)
    scale = oracle.cp_norm(x.weights, x.factors)
    diff = oracle.cp_diff_norm(x.weights, x.factors, res.reduced.weights, res.reduced.factors)
    assert diff <= 1e-6 * scale
    rng = np.random.default_rng(9)
    x = ids.CpTensor(rng.random(7) + 0.5, [rng.standard_normal((d, 7)) for d in (5, 6, 4)])
    res = ids.tensorsketch_id(x, 7, seed=2)
    diff = oracle.cp_diff_norm(x.weights, x.factors, res.reduced.weights, res.reduced.factors)
    assert diff <= 1e-8 * oracle.cp_norm(x.weights, x.factors)


def test_tensor_parameter_validation():
    rng = np.random.default_rng(16)
    x = ids.CpTensor(np.ones(4), [rng.standard_normal((3, 4)), rng.standard_normal((3, 4))])
    with pytest.raises(ValueError):
        ids.tensorsketch_id(x, 5, seed=0)
    with pytest.raises(ValueError):
        ids.tensorsketch_id(x, 2, sketch_dim=9, seed=0)


def test_reduced_preserves_sparsity_pattern():
    rng = np.random.default_rng(15)
    fs = [sp.random_array((10, 6), density=0.3, rng=rng, format="csc") for _ in range(2)]
    x = ids.CpTensor(rng.random(6) + 0.5, fs)
    res = ids.tensorsketch_id(x, 3, seed=4)
    for reduced_f, orig_f in zip(res.reduced.factors, x.factors):
        for t, col in enumerate(res.cols):
            got = reduced_f.toarray()[:, t] != 0
            want = orig_f.toarray()[:, col] != 0
            assert np.array_equal(got, want)


@pytest.mark.parametrize("dims,L", [([30, 20, 10, 8], 5000), ([12, 11], 32768), ([9, 9, 9], 16385),
                                    ([2] * 9, 16), ([40, 30], 65536), ([7, 6, 5], 100_003)])
def test_long_transforms_beyond_the_fused_kernel(dims, L):
    """Sketch lengths whose transform exceeds the fused kernel's shared memory
    (and more than 8 modes) take the per-mode CountSketch + global-memory
    Stockham FFT route (ids_ts_spectral_*); same result as pocketfft."""
    from paper_1901_10559_b200._native import query

    assert not query("ids_tensorsketch_fused_ok", len(dims), L)
    rng = np.random.default_rng(L)
    factors = [rng.standard_normal((d, 5)) for d in dims]
    lam = rng.random(5) + 0.5
    op = ids.TensorSketchOp(dims, L, seed=9)
    want = oracle.OracleTensorSketch(dims, L, seed=9).apply(factors, lam)
    assert relerr_fro(op.apply(factors, lam), want) <= 1e-12
    assert query("ids_tensorsketch_fused_ok", 4, 16384) and query("ids_tensorsketch_fused_ok", 3, 3000)


def test_long_transform_batches_and_weights(monkeypatch):
    # the spectral route in several batches of terms (small work budget),
    # with and without weights, sparse and dense factors
    from paper_1901_10559_b200 import tensorsketch as T

    dims, L, R = [50, 40, 30], 20_000, 23
    M = 65536
    monkeypatch.setattr(T, "SPECTRAL_WORK_BYTES", 3 * 16 * M * 5)  # five terms per batch
    rng = np.random.default_rng(3)
    factors = [rng.standard_normal((d, R)) for d in dims]
    factors[1] = sp.csc_array(factors[1] * (rng.random((dims[1], R)) < 0.3))
    lam = rng.random(R) + 0.5
    op = ids.TensorSketchOp(dims, L, seed=2)
    orc = oracle.OracleTensorSketch(dims, L, seed=2)
    assert relerr_fro(op.apply(factors, lam), orc.apply(factors, lam)) <= 1e-12
    assert relerr_fro(op.apply(factors), orc.apply(factors)) <= 1e-12


# ---- scatter plans (contiguous factor-column reads) vs the gather path ----
def _ts_both(op, factors, weights):
    """Y through the planned kernel and through the plain (gather) entry on
    the same operator and device factors; both (R, L) CUDA tensors."""
    import ctypes

    from paper_1901_10559_b200 import _device
    from paper_1901_10559_b200._native import call, query
    from paper_1901_10559_b200.tensorsketch import factor_to_device, tensorsketch_device

    y_plan = tensorsketch_device(op, factors, weights)
    dev_f = [factor_to_device(f) for f in factors]
    n, L, ncols = len(dev_f), op.out_dim, factors[0].shape[1]
    idx = [m._bucket_index() for m in op.mode_ops]
    fac_p = (ctypes.c_void_p * n)(*[_device.ptr(t) for t in dev_f])
    ord_p = (ctypes.c_void_p * n)(*[_device.ptr(o) for o, _, _ in idx])
    key_p = (ctypes.c_void_p * n)(*[_device.ptr(k) for _, _, k in idx])
    dims = (ctypes.c_int64 * n)(*[int(d) for d in op.mode_dims])
    lds = (ctypes.c_int64 * n)(*[int(t.shape[1]) for t in dev_f])
    w = torch.from_numpy(np.asarray(weights, np.float64)).cuda()
    y = torch.empty((ncols, L), dtype=torch.float64, device="cuda")
    nbytes = query("ids_tensorsketch_workspace_bytes", n, ctypes.addressof(dims), ncols, L)
    ws = _device.workspace(nbytes)
    call("ids_tensorsketch_f64", n, ctypes.addressof(fac_p), ctypes.addressof(dims),
         ctypes.addressof(lds), ncols, ctypes.addressof(ord_p), ctypes.addressof(key_p), L,
         _device.ptr(w), _device.ptr(y), None, _device.ptr(ws), nbytes, _device.stream_ptr())
    return y_plan, y


@pytest.mark.parametrize("dims,L,r", [
    ([10_000] * 4, 16384, 40),      # C5 modes: ~29% of rows collide
    ([1000] * 3, 4096, 50),         # C4 modes
    ([4097, 333, 5], 64, 7),        # heavy collisions: plan falls back for mode 0
    ([1, 2, 3], 8, 3),              # tiny dims
    ([777, 1001], 1000, 9),         # non-power-of-two L (zero-padded transform)
])
def test_scatter_plan_matches_gather_path_bit_for_bit(dims, L, r, monkeypatch):
    from paper_1901_10559_b200 import tensorsketch as tsmod

    monkeypatch.setattr(tsmod, "SCATTER_MIN_DIM", 1)  # plans for every mode
    monkeypatch.setattr(tsmod, "USE_SPLIT", False)  # the one-CTA-per-term kernel's plans
    rng = np.random.default_rng(sum(dims) + L)
    factors = [rng.standard_normal((d, r)) for d in dims]
    weights = rng.random(r) + 0.5
    op = ids.TensorSketchOp(dims, L, seed=3)
    y_plan, y_gather = _ts_both(op, factors, weights)
    assert torch.equal(y_plan, y_gather)
    want = oracle.tensorsketch_apply(
        oracle.OracleTensorSketch(dims, L, seed=3).mode_ops, L, factors, weights)
    assert relerr_fro(y_plan.t().cpu().numpy(), want) <= 1e-12


def test_scatter_plan_ranks_and_slots():
    """The plan's per-row code/rank layout against numpy: rank = position
    among the rows of the same bucket in increasing row order; every row
    with rank >= 1 owns one stash slot inside its rank's range."""
    from paper_1901_10559_b200 import _device  # noqa: F401

    op = ids.CountSketchOp(5000, 3000, seed=11)
    plan = op._ts_plan().cpu().numpy().view(np.int32)
    hdr = plan[:168]
    valid, maxr, nstash = hdr[0], hdr[1], hdr[2]
    off = hdr[4 + 64 + 64:]
    stride = (5000 + 3) & ~3
    code = plan[168:168 + 5000]
    slot = plan[168 + stride:168 + stride + 5000]
    b = op.bucket
    assert np.array_equal(np.where(code >= 0, code, ~code), b)
    assert np.array_equal(code >= 0, op.sign > 0)
    rank = np.zeros(5000, np.int64)
    seen = {}
    for i in range(5000):
        rank[i] = seen.get(b[i], 0)
        seen[b[i]] = rank[i] + 1
    assert valid == 1 and maxr == rank.max() and nstash == (rank >= 1).sum()
    assert np.all(slot[rank == 0] == -1)
    for rr in range(1, maxr + 1):
        s = np.sort(slot[rank == rr])
        assert np.array_equal(s, np.arange(off[rr], off[rr + 1]))


def test_colnorm_epilogue_feeds_cpqr():
    """The fused kernel's ||Y[:, r]||^2 epilogue (fixed-order: run-to-run
    identical) equals the norms of the written sketch, and the CPQR that
    takes it (ids_cpqr_trunc_norms_f64, no initial norm pass) picks the
    same pivots and R as the one that computes its own (linalg.py:97)."""
    from paper_1901_10559_b200.linalg import device_cpqr

    rng = np.random.default_rng(21)
    w, fac = _near_dup_cp(rng, [3000] * 3, 600, 12, 1e-3)
    x = ids.CpTensor(w, fac)
    op = ids.TensorSketchOp(x.mode_dims, 4096, seed=3)
    y, nrm = op.apply_device(x.factors, x.weights, norms=True)
    y2, nrm2 = op.apply_device(x.factors, x.weights, norms=True)
    assert torch.equal(nrm, nrm2) and torch.equal(y, y2)
    ref = (y * y).sum(dim=1)
    assert float(((nrm - ref).abs() / ref).max()) <= 1e-13
    a = device_cpqr(y, 4096, 600, 12)
    b = device_cpqr(y, 4096, 600, 12, colnorm2=nrm)
    assert torch.equal(a.perm[:12], b.perm[:12])
    assert float((a.rtop - b.rtop).abs().max() / a.rtop.abs().max()) <= 1e-12
    want = oracle.cpqr(y.t().cpu().numpy(), 12)
    assert np.array_equal(b.perm[:12].cpu().numpy(), want.perm[:12])


@pytest.mark.parametrize("L", [64, 4096, 16384, 20000])
def test_sparse_factors_native_path_matches_dense(L):
    """CSC factors are CountSketched from their sparse arrays (never
    densified): the sketch is bit-identical to the same factors passed dense
    (one-CTA-per-term kernel), agrees to rounding where the order of the
    CountSketch sums differs (split-spectrum kernel: buckets b and b + L/2
    folded row by row on the dense path, bucket sums folded on the sparse
    one; spectral route), and matches the oracle (reference sketch.py:175
    sketches CSC directly)."""
    rng = np.random.default_rng(L)
    dims = [5000, 300, 7000]
    fs = [sp.random_array((d, 12), density=0.02, rng=rng, format="csc") for d in dims]
    fs[1] = fs[1].toarray()  # mixed: one dense mode
    lam = rng.random(12) + 0.5
    op = ids.TensorSketchOp(dims, L, seed=4)
    y_sparse = op.apply(fs, lam)
    y_dense = op.apply([f.toarray() if sp.issparse(f) else f for f in fs], lam)
    from paper_1901_10559_b200.tensorsketch import uses_split_kernel

    if L <= 16384 and not uses_split_kernel(len(dims), L):
        assert np.array_equal(y_sparse, y_dense)
    else:
        assert relerr_fro(y_sparse, y_dense) <= 1e-14
    want = oracle.OracleTensorSketch(dims, L, seed=4).apply(fs, lam)
    assert relerr_fro(y_sparse, want) <= 1e-12

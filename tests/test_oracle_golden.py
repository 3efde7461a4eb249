"""Pin the CPU oracle against golden vectors produced by the real reference
(tests/golden/make_golden.py).  CPU only."""

import hashlib

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from oracle.cs_hash import countsketch_dense_sequential

from conftest import relerr_fro


def _digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_hash_small_bit_exact(golden):
    data, man = golden
    for case in man["hash_small"]:
        op = oracle.OracleCountSketch(
            case["in_dim"], case["out_dim"], case["seed"], case["surjective"]
        )
        assert np.array_equal(op.bucket, data[f"hash{case['id']}_bucket"]), case
        assert np.array_equal(op.sign, data[f"hash{case['id']}_sign"]), case


@pytest.mark.parametrize("which", ["small", "large"])
def test_hash_digests(golden, which):
    _, man = golden
    for case in man["hash_digest"]:
        big = case["in_dim"] * (1 if case["mode"] is None else 1) > 3_000_000
        if (which == "large") != big:
            continue
        op = oracle.OracleCountSketch(
            case["in_dim"], case["out_dim"], case["seed"], case["surjective"],
            mode=case["mode"],
        )
        assert _digest(op.bucket, op.sign) == case["sha256"], case


def test_hash_matches_numpy_generator_directly():
    # random shapes against numpy's own Generator (the third-party source)
    rng = np.random.default_rng(77)
    for _ in range(40):
        I = int(rng.integers(1, 5000))
        L = int(rng.integers(1, I + 1))
        surj = bool(rng.integers(0, 2))
        seed = int(rng.integers(0, 2**31))
        g = np.random.default_rng(seed)
        if surj:
            tail = g.integers(0, L, size=I - L)
            b = g.permutation(np.concatenate([np.arange(L, dtype=np.int64), tail]))
        else:
            b = g.integers(0, L, size=I)
        s = g.integers(0, 2, size=I).astype(np.float64) * 2.0 - 1.0
        op = oracle.OracleCountSketch(I, L, seed, surj)
        assert np.array_equal(op.bucket, b)
        assert np.array_equal(op.sign, s)


def test_stream32_matches_numpy():
    st, inc = oracle.seed_state(123)
    ours = oracle.pcg64_stream32(st, inc, 1001)
    g = np.random.Generator(np.random.PCG64(123))
    want = g.integers(0, 2**32, size=1001, dtype=np.uint64).astype(np.uint32)
    assert np.array_equal(ours, want)


def test_sketch_dense_golden(golden):
    data, man = golden
    for case in man["sketch_dense"]:
        n = case["id"]
        op = oracle.OracleCountSketch(
            case["in_dim"], case["out_dim"], case["seed"], case["surjective"]
        )
        a = data[f"sd{n}_a"]
        y = op.apply(a)
        assert np.array_equal(y, data[f"sd{n}_y"])
        # the sequential C restatement reproduces scipy's summation order bit for bit
        y2 = countsketch_dense_sequential(a, op.bucket, op.sign, case["out_dim"])
        assert np.array_equal(y2, data[f"sd{n}_y"])


def test_sketch_csr_golden(golden):
    data, man = golden
    for case in man["sketch_csr"]:
        n = case["id"]
        a = sp.csr_array(
            (data[f"sc{n}_data"], data[f"sc{n}_indices"], data[f"sc{n}_indptr"]),
            shape=(case["in_dim"], case["cols"]),
        )
        op = oracle.OracleCountSketch(
            case["in_dim"], case["out_dim"], case["seed"], case["surjective"]
        )
        # reference canonicalizes to CSC first (linalg.py:39-53)
        assert np.array_equal(op.apply(sp.csc_array(a)), data[f"sc{n}_y"])


def test_tensorsketch_golden(golden):
    data, man = golden
    for case in man["tensorsketch"]:
        n = case["id"]
        factors = [data[f"ts{n}_f{m}"] for m in range(len(case["dims"]))]
        ts = oracle.OracleTensorSketch(case["dims"], case["out_dim"], case["seed"])
        y = ts.apply(factors, data[f"ts{n}_w"])
        assert np.array_equal(y, data[f"ts{n}_y"])


def test_matrix_id_golden(golden):
    data, man = golden
    for case in man["matrix_id"]:
        n = case["id"]
        d = oracle.matrix_id(data[f"mid{n}_y"], case["rank"])
        assert np.array_equal(d.cols, data[f"mid{n}_cols"])
        assert np.array_equal(d.coeffs, data[f"mid{n}_coeffs"])
        assert d.numerical_rank == case["numerical_rank"]
        assert d.rank_deficient == case["rank_deficient"]


def test_countsketch_id_golden(golden):
    data, man = golden
    a = data["csid_a"]
    for case in man["countsketch_id"]:
        s = case["seed"]
        d = oracle.countsketch_id(a, case["rank"], case["sketch_dim"], seed=s)
        assert np.array_equal(d.sketch, data[f"csid{s}_y"])
        assert np.array_equal(d.cols, data[f"csid{s}_cols"])
        assert relerr_fro(d.coeffs, data[f"csid{s}_coeffs"]) == 0.0
    a_sp = sp.csr_array(
        (data["csid_sp_data"], data["csid_sp_indices"], data["csid_sp_indptr"]),
        shape=(3000, 120),
    )
    d = oracle.countsketch_id(sp.csc_array(a_sp), 12, 50, seed=21)
    assert np.array_equal(d.cols, data["csid_sp_cols"])
    assert np.array_equal(d.coeffs, data["csid_sp_coeffs"])


def test_tensorsketch_id_golden(golden):
    data, man = golden
    case = man["tensorsketch_id"][0]
    factors = [data[f"tsid_f{m}"] for m in range(len(case["dims"]))]
    d, nw = oracle.tensorsketch_id(
        data["tsid_w"], factors, case["rank"], case["sketch_dim"], seed=case["seed"]
    )
    assert np.array_equal(d.cols, data["tsid_cols"])
    assert np.array_equal(d.coeffs, data["tsid_coeffs"])
    assert np.array_equal(nw, data["tsid_new_weights"])


def test_error_estimates_golden(golden):
    """The reference's error metric (estimators.py, bench.py:137-145) restated."""
    data, man = golden
    a = data["csid_a"]
    a_sp = sp.csr_array(
        (data["csid_sp_data"], data["csid_sp_indices"], data["csid_sp_indptr"]),
        shape=(3000, 120),
    )
    for case in man["error_estimates"]:
        if case["case"] == "csid":
            s = case["seed"]
            assert oracle.derive_seed(s, 0xE57) == case["est_seed"]
            ap, adj = oracle.id_residual_operator(a, data[f"csid{s}_cols"], data[f"csid{s}_coeffs"])
            v = oracle.est_spectral_norm(ap, adj, a.shape[1], seed=case["est_seed"])
        elif case["case"] == "csid_sp":
            assert oracle.derive_seed(21, 0xE57) == case["est_seed"]
            ap, adj = oracle.id_residual_operator(a_sp, data["csid_sp_cols"], data["csid_sp_coeffs"])
            v = oracle.est_spectral_norm(ap, adj, a_sp.shape[1], seed=case["est_seed"])
        else:
            ap, adj = oracle.matrix_operator(a)
            v = oracle.est_spectral_norm(ap, adj, a.shape[1], iters=case["iters"],
                                         probes=case["probes"], seed=case["est_seed"])
        assert v == case["value"], case
    tcase = man["tensorsketch_id"][0]
    factors = [data[f"tsid_f{m}"] for m in range(len(tcase["dims"]))]
    w = data["tsid_w"]
    cols = data["tsid_cols"]
    err = oracle.cp_diff_norm(w, factors, data["tsid_new_weights"], [f[:, cols] for f in factors])
    assert abs(err - tcase["cp_diff_norm"]) <= 1e-12 * tcase["cp_norm"]
    assert abs(oracle.cp_norm(w, factors) - tcase["cp_norm"]) <= 1e-12 * tcase["cp_norm"]

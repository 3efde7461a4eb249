"""The C-ABI library loads and exports every symbol include/idsketch_b200.h
declares (no compute: runs without a GPU)."""

import ctypes
import os
import re

from paper_1901_10559_b200 import _native

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "idsketch_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(ids_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


def test_header_declares_functions():
    names = declared_functions()
    assert "ids_countsketch_hash" in names
    assert "ids_countsketch_dense_f64" in names
    assert "ids_tensorsketch_f64" in names
    assert "ids_cpqr_trunc_f64" in names
    assert len(names) >= 18


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert set(declared_functions()) == set(_native.SIGNATURES)


def test_workspace_queries_without_gpu():
    # size queries are pure host arithmetic
    assert _native.query("ids_hash_workspace_bytes", 1_000_000, 100, 1) > 8_000_000
    assert _native.query("ids_hash_workspace_bytes", 1000, 10, 0) > 0
    assert _native.query("ids_cpqr_workspace_bytes", 100, 2000, 20) > 100 * 20 * 8
    assert _native.query("ids_bucket_index_workspace_bytes", 10_000, 40) > 80_000
    assert _native.query("ids_id_coeffs_workspace_bytes", 20, 2000) >= 20 * 1980 * 8
    assert _native.load().ids_version() == 1


def test_shared_object_is_sm100a():
    # the fatbin inside the library must carry sm_100a SASS
    data = open(_native.LIB_PATH, "rb").read()
    assert b"sm_100a" in data

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun)")


@pytest.fixture(scope="session")
def golden():
    data = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    with open(os.path.join(GOLDEN_DIR, "manifest.json")) as fh:
        manifest = json.load(fh)
    return data, manifest


def relerr_fro(got, want):
    want = np.asarray(want)
    den = np.linalg.norm(want)
    return np.linalg.norm(np.asarray(got) - want) / (den if den > 0 else 1.0)


def khatri_rao(mats):
    """Columnwise Kronecker product, first matrix slowest (reference conftest.py:13-19)."""
    out = np.asarray(mats[0])
    for m in mats[1:]:
        out = (out[:, None, :] * np.asarray(m)[None, :, :]).reshape(-1, out.shape[1])
    return out


def dense_countsketch(bucket, sign, out_dim):
    s = np.zeros((out_dim, bucket.size))
    s[bucket, np.arange(bucket.size)] = sign
    return s

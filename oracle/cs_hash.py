"""ctypes front-end of ``hash_oracle.c`` -- TEST INFRASTRUCTURE ONLY.

Restates reference ``pkg/src/idsketch/sketch.py:77-84`` (bucket and sign
draws of ``CountSketchOp``) and ``sketch.py:143-150`` (per-mode seeding of
``TensorSketchOp`` via ``SeedSequence([entropy, n])``).
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libidsketch_oracle.so")
_lib = None


def build():
    """Compile the C oracle (gcc) into oracle/_build/."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        u64, i64 = ctypes.c_uint64, ctypes.c_int64
        lib.oracle_countsketch_hash.argtypes = [
            u64, u64, u64, u64, i64, i64, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
        ]
        lib.oracle_countsketch_hash.restype = ctypes.c_int
        lib.oracle_pcg64_stream32.argtypes = [u64, u64, u64, u64, i64, ctypes.c_void_p]
        lib.oracle_pcg64_stream32.restype = ctypes.c_int
        lib.oracle_countsketch_dense.argtypes = [
            ctypes.c_void_p, i64, i64, i64, ctypes.c_void_p, ctypes.c_void_p, i64,
            ctypes.c_void_p,
        ]
        lib.oracle_countsketch_dense.restype = ctypes.c_int
        _lib = lib
    return _lib


def seed_state(seed, mode=None):
    """(state, inc) of the fresh PCG64 numpy builds for ``default_rng(seed)``
    (``sketch.py:77``) or, with ``mode=n``, for ``SeedSequence([seed, n])``
    (``sketch.py:148``)."""
    if mode is not None:
        ss = np.random.SeedSequence([int(seed), int(mode)])
    elif isinstance(seed, np.random.SeedSequence):
        ss = seed
    else:
        ss = np.random.SeedSequence(seed)
    st = np.random.PCG64(ss).state["state"]
    return int(st["state"]), int(st["inc"])


def _split(v):
    return (v >> 64) & 0xFFFFFFFFFFFFFFFF, v & 0xFFFFFFFFFFFFFFFF


def countsketch_hash(in_dim, out_dim, state, inc, surjective):
    """bucket int64[in_dim], sign float64[in_dim], draws (A, B, signs)."""
    lib = _load()
    bucket = np.empty(in_dim, dtype=np.int64)
    sign = np.empty(in_dim, dtype=np.float64)
    draws = np.zeros(3, dtype=np.int64)
    sh, sl = _split(state)
    ih, il = _split(inc)
    rc = lib.oracle_countsketch_hash(
        sh, sl, ih, il, int(in_dim), int(out_dim), int(bool(surjective)),
        bucket.ctypes.data, sign.ctypes.data, draws.ctypes.data,
    )
    if rc != 0:
        raise ValueError("bad CountSketch hash arguments")
    return bucket, sign, draws


def pcg64_stream32(state, inc, n):
    lib = _load()
    out = np.empty(n, dtype=np.uint32)
    sh, sl = _split(state)
    ih, il = _split(inc)
    lib.oracle_pcg64_stream32(sh, sl, ih, il, int(n), out.ctypes.data)
    return out


def countsketch_dense_sequential(a, bucket, sign, out_dim):
    """Sequential (scipy-order) S @ A for a C-ordered dense A."""
    lib = _load()
    a = np.ascontiguousarray(a, dtype=np.float64)
    bucket = np.ascontiguousarray(bucket, dtype=np.int64)
    sign = np.ascontiguousarray(sign, dtype=np.float64)
    y = np.empty((out_dim, a.shape[1]), dtype=np.float64)
    lib.oracle_countsketch_dense(
        a.ctypes.data, a.shape[0], a.shape[1], a.shape[1],
        bucket.ctypes.data, sign.ctypes.data, int(out_dim), y.ctypes.data,
    )
    return y

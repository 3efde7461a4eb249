"""CPU oracle for the CountSketch / TensorSketch ID hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline.  The product package (``paper_1901_10559_b200``) never
imports it and has no CPU fallback.

Contents
--------
* ``hash_oracle.c`` (built to ``oracle/_build/libidsketch_oracle.so`` by
  ``oracle/Makefile``): plain-C restatement of the PCG64 / Lemire /
  Fisher-Yates draw sequence behind ``CountSketchOp.__init__``
  (reference ``pkg/src/idsketch/sketch.py:77-84``).
* ``estimators.py``: the reference's error metric for matrix trials
  (``estimators.py:26-121``, ``bench.py:116-145``).
* ``dcpqr.py``: one rank's share of the column-distributed CPQR (the
  interface of ``distributed.DeviceCpqrShard``), for gloo tests of the host
  driver.
* ``port.py``: numpy/scipy restatement of the reference's sketch + ID path
  (``sketch.py:116-186``, ``linalg.py:76-147``, ``matrix_id.py:56-182``,
  ``cp_tensor.py:215-276``), calling the same third-party kernels the
  reference calls (scipy sparse products, pocketfft, LAPACK dgeqp3/dtrtrs).

Parity pin: the oracle is checked against golden vectors produced by the
real reference package (``tests/golden/make_golden.py``) in
``tests/test_oracle_golden.py``.
"""

from .cs_hash import countsketch_hash, pcg64_stream32, seed_state
from .dcpqr import OracleCpqrShard
from .estimators import derive_seed, est_spectral_norm, id_residual_operator, matrix_operator
from .port import (
    OracleCountSketch,
    OracleTensorSketch,
    coeffs_from_pivoted,
    cp_gram,
    countsketch_id,
    cp_diff_norm,
    cp_norm,
    cpqr,
    cs_apply,
    matrix_id,
    tensorsketch_apply,
    tensorsketch_id,
    ts_new_weights,
)

__all__ = [
    "OracleCountSketch",
    "OracleCpqrShard",
    "OracleTensorSketch",
    "coeffs_from_pivoted",
    "cp_gram",
    "countsketch_hash",
    "countsketch_id",
    "cp_diff_norm",
    "cp_norm",
    "cpqr",
    "cs_apply",
    "derive_seed",
    "est_spectral_norm",
    "id_residual_operator",
    "matrix_operator",
    "matrix_id",
    "pcg64_stream32",
    "seed_state",
    "tensorsketch_apply",
    "tensorsketch_id",
    "ts_new_weights",
]

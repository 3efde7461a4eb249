"""B200-native CountSketch / TensorSketch interpolative decomposition.

Drop-in for the hot path of the reference package ``idsketch`` (arXiv
1901.10559): the public names below keep the reference's signatures,
defaults, return layout and exceptions (reference ``pkg/src/idsketch/
__init__.py:9-86``), restricted to the CountSketch matrix ID and TensorSketch
tensor ID path.  All compute runs in hand-written sm_100a kernels reached
through the C ABI of ``include/idsketch_b200.h`` (``libidsketch_b200.so``);
there is no CPU fallback.
"""

from .cp_tensor import (
    CpTensor,
    TensorIdGraph,
    TensorIdResult,
    check_tensor_id_args,
    cp_diff_norm,
    cp_norm,
    gram_hadamard,
    tensor_id_from_sketch,
    tensorsketch_id,
)
from .errors import SingularTriangleError
from .estimators import (
    NormEstimate,
    derive_seed,
    est_spectral_norm,
    id_residual_operator,
    matrix_operator,
)
from .linalg import DEFAULT_RANK_TOL, PivotedQr, cpqr, triangular_solve
from .matrix_id import (
    InterpolativeDecomposition,
    check_matrix_id_args,
    countsketch_id,
    matrix_id,
    matrix_sketch,
)
from .mmio import (
    load_cp_dir,
    read_matrix_market,
    read_matrix_market_device,
    save_cp_dir,
    write_matrix_market,
)
from .sketch import (
    CountSketchOp,
    NondeterministicSketchWarning,
    TensorSketchOp,
    set_sparse_sketch_mode,
)

__version__ = "0.1.0"

__all__ = [
    "CountSketchOp",
    "CpTensor",
    "DEFAULT_RANK_TOL",
    "InterpolativeDecomposition",
    "NondeterministicSketchWarning",
    "NormEstimate",
    "PivotedQr",
    "SingularTriangleError",
    "TensorIdGraph",
    "TensorIdResult",
    "TensorSketchOp",
    "check_matrix_id_args",
    "check_tensor_id_args",
    "countsketch_id",
    "cp_diff_norm",
    "cp_norm",
    "cpqr",
    "derive_seed",
    "est_spectral_norm",
    "gram_hadamard",
    "id_residual_operator",
    "load_cp_dir",
    "matrix_id",
    "matrix_operator",
    "matrix_sketch",
    "read_matrix_market",
    "read_matrix_market_device",
    "save_cp_dir",
    "set_sparse_sketch_mode",
    "tensor_id_from_sketch",
    "tensorsketch_id",
    "triangular_solve",
    "write_matrix_market",
]

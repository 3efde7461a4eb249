"""ctypes binding of the C ABI in include/idsketch_b200.h (libidsketch_b200.so).

This is the only way the package reaches compute: there is no CPU fallback.
If the shared library is missing the import fails loudly; build it with
``python -c "import __graft_entry__; __graft_entry__.build()"`` (or ``make -C
paper_1901_10559_b200/csrc``).
"""

import ctypes
import os

from .errors import SingularTriangleError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libidsketch_b200.so")

IDS_OK, IDS_EINVAL, IDS_ENONFINITE, IDS_ESINGULAR, IDS_ECUDA, IDS_EWORKSPACE, IDS_ERETRY = range(7)
IDS_ROW_MAJOR, IDS_COL_MAJOR = 0, 1
IDS_FLAG_ORDERED = 1
IDS_FLAG_DETERMINISTIC = 2

_c_i64, _c_u64, _c_int, _c_dbl = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
_c_sz, _c_p = ctypes.c_size_t, ctypes.c_void_p

# name -> (restype, argtypes)
SIGNATURES = {
    "ids_last_error": (ctypes.c_char_p, []),
    "ids_version": (_c_int, []),
    "ids_launch_count": (_c_i64, []),
    "ids_probe_fp64_tflops": (_c_dbl, [_c_p]),
    "ids_hash_workspace_bytes": (_c_sz, [_c_i64, _c_i64, _c_int]),
    "ids_countsketch_hash": (
        _c_int,
        [_c_u64, _c_u64, _c_u64, _c_u64, _c_i64, _c_i64, _c_int, _c_p, _c_p, _c_p, _c_p, _c_sz,
         _c_p],
    ),
    "ids_countsketch_hash_dev": (
        _c_int, [_c_p, _c_i64, _c_i64, _c_int, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]
    ),
    "ids_bucket_index_workspace_bytes": (_c_sz, [_c_i64, _c_i64]),
    "ids_bucket_index": (
        _c_int, [_c_p, _c_p, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]
    ),
    "ids_countsketch_dense_workspace_bytes": (_c_sz, [_c_i64, _c_i64, _c_i64, _c_int]),
    "ids_countsketch_dense_f64": (
        _c_int,
        [_c_p, _c_i64, _c_i64, _c_i64, _c_int, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_i64,
         _c_p, _c_int, _c_int, _c_p, _c_p, _c_sz, _c_p],
    ),
    "ids_dense_has_nonfinite": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_int, _c_p, _c_p]),
    "ids_countsketch_csc_workspace_bytes": (_c_sz, [_c_i64, _c_i64]),
    "ids_countsketch_csc_f64": (
        _c_int,
        [_c_p, _c_int, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_i64,
         _c_p, _c_int, _c_p, _c_p, _c_sz, _c_p],
    ),
    "ids_values_has_nonfinite": (_c_int, [_c_p, _c_i64, _c_p, _c_p]),
    "ids_countsketch_csr_workspace_bytes": (_c_sz, [_c_i64, _c_i64, _c_i64, _c_i64]),
    "ids_countsketch_csr_f64": (
        _c_int,
        [_c_p, _c_int, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p,
         _c_p, _c_i64, _c_p, _c_int, _c_int, _c_p, _c_p, _c_sz, _c_p],
    ),
    "ids_tensorsketch_workspace_bytes": (_c_sz, [_c_int, _c_p, _c_i64, _c_i64]),
    "ids_tensorsketch_fused_ok": (_c_int, [_c_int, _c_i64]),
    "ids_tensorsketch_f64": (
        _c_int,
        [_c_int, _c_p, _c_p, _c_p, _c_i64, _c_p, _c_p, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_sz,
         _c_p],
    ),
    "ids_ts_mode_plan_bytes": (_c_sz, [_c_i64]),
    "ids_ts_mode_plan": (_c_int, [_c_p, _c_p, _c_p, _c_i64, _c_i64, _c_p, _c_sz, _c_p]),
    "ids_tensorsketch_planned_f64": (
        _c_int,
        [_c_int, _c_p, _c_p, _c_p, _c_i64, _c_p, _c_p, _c_p, _c_i64, _c_p, _c_p, _c_p, _c_p,
         _c_sz, _c_p],
    ),
    "ids_tensorsketch_split_ok": (_c_int, [_c_int, _c_i64]),
    "ids_ts_spectral_len": (_c_i64, [_c_int, _c_i64]),
    "ids_ts_spectral_mode_f64": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_int, _c_p]),
    "ids_ts_spectral_pair_f64": (
        _c_int, [_c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_int, _c_p]
    ),
    "ids_ts_spectral_finish_f64": (_c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p]),
    "ids_ts_split_plan_bytes": (_c_sz, [_c_i64, _c_i64]),
    "ids_ts_split_plan": (_c_int, [_c_p, _c_p, _c_i64, _c_i64, _c_p, _c_sz, _c_p]),
    "ids_tensorsketch_split_f64": (
        _c_int, [_c_int, _c_p, _c_p, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_p, _c_p, _c_p]
    ),
    "ids_cpqr_workspace_bytes": (_c_sz, [_c_i64, _c_i64, _c_i64]),
    "ids_cpqr_trunc_f64": (
        _c_int,
        [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_dbl, _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p],
    ),
    "ids_cpqr_trunc_norms_f64": (
        _c_int,
        [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_dbl, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_sz,
         _c_p],
    ),
    "ids_id_coeffs_workspace_bytes": (_c_sz, [_c_i64, _c_i64]),
    "ids_id_coeffs_f64": (
        _c_int,
        [_c_p, _c_p, _c_i64, _c_i64, _c_dbl, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p],
    ),
    "ids_triangular_solve_f64": (
        _c_int, [_c_p, _c_p, _c_i64, _c_i64, _c_int, _c_p, _c_p, _c_p]
    ),
    "ids_set_hash_grid_cap": (None, [_c_int]),
    "ids_set_hash_stages": (None, [_c_int, _c_i64]),
    "ids_mm_info": (_c_int, [ctypes.c_char_p, _c_p, _c_p, _c_p, _c_p]),
    "ids_mm_read": (_c_int, [ctypes.c_char_p, _c_int, _c_p, _c_p, _c_p, _c_i64, _c_p]),
    "ids_dcpqr_workspace_bytes": (_c_sz, [_c_i64, _c_i64, _c_i64]),
    "ids_dcpqr_init_f64": (
        _c_int, [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_sz, _c_p]
    ),
    "ids_dcpqr_pivot_f64": (
        _c_int,
        [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_p,
         _c_p, _c_sz, _c_p],
    ),
    "ids_dcpqr_step_f64": (
        _c_int,
        [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_sz,
         _c_p],
    ),
    "ids_dcpqr_select_f64": (_c_int, [_c_p, _c_i64, _c_i64, _c_p, _c_p]),
    "ids_dcpqr_pivot_dev_f64": (
        _c_int,
        [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_sz, _c_p],
    ),
    "ids_dcpqr_step_dev_f64": (
        _c_int,
        [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_sz,
         _c_p],
    ),
    "ids_dcpqr_select_pivot_f64": (
        _c_int,
        [_c_p, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_p, _c_p,
         _c_sz, _c_p],
    ),
    "ids_dcpqr_results_f64": (
        _c_int, [_c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p]
    ),
    "ids_dense_gemv_workspace_bytes": (_c_sz, [_c_i64, _c_i64, _c_int, _c_int]),
    "ids_dense_gemv_f64": (
        _c_int,
        [_c_p, _c_i64, _c_i64, _c_i64, _c_int, _c_int, _c_p, _c_p, _c_p, _c_sz, _c_p],
    ),
    "ids_csr_spmv_f64": (
        _c_int, [_c_p, _c_int, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p]
    ),
    "ids_csr_transpose_workspace_bytes": (_c_sz, [_c_i64, _c_i64, _c_i64]),
    "ids_csr_transpose_f64": (
        _c_int,
        [_c_p, _c_int, _c_p, _c_p, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_sz, _c_p],
    ),
}

_lib = None


def load():
    """Load libidsketch_b200.so (in-tree) and declare every C-ABI signature."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the B200 kernels are not built (no CPU fallback); "
            "run __graft_entry__.build()"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc, what=""):
    """Map a C-ABI status to the reference's exception types."""
    if rc == IDS_OK:
        return
    msg = load().ids_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc in (IDS_EINVAL, IDS_ENONFINITE):
        raise ValueError(text)
    if rc == IDS_ESINGULAR:
        raise SingularTriangleError(text)
    raise RuntimeError(text)


def call(name, *args):
    """Call a C-ABI function that returns a status code; raise on failure."""
    rc = getattr(load(), name)(*args)
    check(rc, name)


def query(name, *args):
    return int(getattr(load(), name)(*args))

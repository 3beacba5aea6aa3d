"""ctypes binding of ``libcpfit_b200.so`` (the C-ABI in include/cpfit_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, the kernel entry points raise instead of computing.
"""

from __future__ import annotations

import ctypes
import os

from .exceptions import NumericalError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcpfit_b200.so")

OK = 0
EINVAL = 1
ECUDA = 2
ESINGULAR = 3
EEMPTYROW = 4
ENEGWEIGHT = 5
ENONFINITE = 6
ENOMEM = 7

F64 = 0
F32 = 1

# every entry point the header declares (checked by tests/test_abi.py)
SYMBOLS = (
    "cpfit_version", "cpfit_last_error",
    "cpfit_pattern_create", "cpfit_pattern_create_coords", "cpfit_pattern_destroy",
    "cpfit_pattern_info", "cpfit_pattern_coords", "cpfit_pattern_set_task_size",
    "cpfit_pattern_mode_group", "cpfit_pattern_mode_stats", "cpfit_permute_values",
    "cpfit_tttp", "cpfit_mttkrp", "cpfit_gram", "cpfit_solve_factor",
    "cpfit_tttp_axpby", "cpfit_sample", "cpfit_pattern_parent_index", "cpfit_gather_values",
    "cpfit_reduce", "cpfit_sgd_update", "cpfit_ccd_step", "cpfit_probe_gather",
    "cpfit_solve_rows", "cpfit_dense_reduce", "cpfit_khatri_rao", "cpfit_als_update",
    "cpfit_ccd_fold", "cpfit_ccd_finalize", "cpfit_check_finite",
    "cpfit_tttp_host", "cpfit_tttp_subst", "cpfit_axpby", "cpfit_spd_inverse_rows",
    "cpfit_batched_symv", "cpfit_tttp_loss", "cpfit_loss_eval", "cpfit_ccd_gen_weights",
    "cpfit_ccd_gen_update", "cpfit_ccd_gen_model", "cpfit_from_coords",
    "cpfit_tttp_host_async", "cpfit_event_wait", "cpfit_copy_to_host",
    "cpfit_ccsr_spmm", "cpfit_pairwise_tttp", "cpfit_pairwise_fold_sum",
    "cpfit_dense_mttkrp", "cpfit_dense_xc", "cpfit_dense_gram", "cpfit_probe_l2_read",
    "cpfit_gram_matvec", "cpfit_cg_rows_init", "cpfit_cg_rows_step",
    "cpfit_pattern_destroy_async",
)

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int
_PP = ctypes.POINTER(ctypes.c_void_p)

_lib = None


class CpfitError(RuntimeError):
    """Unexpected failure inside the CUDA library (launch / runtime errors)."""


def load(path: str | None = None):
    """Load the shared library and declare the C signatures."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("CPFIT_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")
    L = ctypes.CDLL(path)
    L.cpfit_version.restype = ctypes.c_char_p
    L.cpfit_last_error.restype = ctypes.c_char_p
    sig = {
        "cpfit_pattern_create": [_int, ctypes.POINTER(_i64), _i64, _vp, _vp, ctypes.POINTER(_vp)],
        "cpfit_pattern_create_coords": [_int, ctypes.POINTER(_i64), _i64, _PP, _vp,
                                        ctypes.POINTER(_vp)],
        "cpfit_pattern_destroy": [_vp],
        "cpfit_pattern_destroy_async": [_vp, _vp],
        "cpfit_pattern_info": [_vp, ctypes.POINTER(_int), ctypes.POINTER(_i64)],
        "cpfit_pattern_coords": [_vp, _int, ctypes.POINTER(_vp)],
        "cpfit_pattern_set_task_size": [_vp, _i64],
        "cpfit_pattern_mode_group": [_vp, _int, _vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp)],
        "cpfit_pattern_mode_stats": [_vp, _int, _vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                     ctypes.POINTER(_i64)],
        "cpfit_permute_values": [_vp, _int, _int, _vp, _vp, _vp],
        "cpfit_tttp": [_vp, _int, _int, _vp, _PP, _vp, _vp],
        "cpfit_mttkrp": [_vp, _int, _int, _int, _vp, _int, _PP, _vp, _vp],
        "cpfit_gram": [_vp, _int, _int, _int, _vp, _int, _PP, _vp, _vp],
        "cpfit_solve_factor": [_vp, _int, _int, _int, _vp, _int, _PP, _vp, ctypes.c_double,
                               _vp, _vp, ctypes.POINTER(_i64), _vp],
        "cpfit_tttp_axpby": [_vp, _int, _int, _vp, _PP, ctypes.c_double, ctypes.c_double,
                             _vp, _vp],
        "cpfit_sample": [_vp, ctypes.c_uint64, ctypes.c_uint64, _i64, ctypes.c_double, _vp,
                         ctypes.POINTER(_vp)],
        "cpfit_pattern_parent_index": [_vp, ctypes.POINTER(_vp)],
        "cpfit_gather_values": [_int, _i64, _vp, _vp, _vp, _vp],
        "cpfit_reduce": [_int, _int, _i64, _vp, _vp, ctypes.POINTER(ctypes.c_double), _vp],
        "cpfit_sgd_update": [_int, _i64, _vp, _vp, ctypes.c_double, ctypes.c_double, _vp,
                             ctypes.POINTER(_int), _vp],
        "cpfit_ccd_step": [_vp, _int, _PP, _vp, _int, _PP, _PP, ctypes.c_double, _vp, _vp],
        "cpfit_tttp_host": [_vp, _int, _int, _vp, _PP, _vp, _vp, _i64, _vp],
        "cpfit_tttp_host_async": [_vp, _int, _int, _vp, _PP, _vp, _vp, _i64,
                                  ctypes.POINTER(_vp), _vp],
        "cpfit_event_wait": [_vp, _int],
        "cpfit_copy_to_host": [_i64, _vp, _vp, _vp],
        "cpfit_ccsr_spmm": [_i64, _vp, _vp, _vp, _vp, _int, _vp, _vp],
        "cpfit_pairwise_tttp": [_i64, _int, _int, _PP, _PP, _vp, _vp, _vp],
        "cpfit_pairwise_fold_sum": [_i64, _int, _int, _PP, _PP, _vp, _vp, _i64, _vp, _vp],
        "cpfit_tttp_subst": [_vp, _int, _int, _vp, _PP, _PP, _vp, _vp],
        "cpfit_axpby": [_int, _i64, ctypes.c_double, _vp, ctypes.c_double, _vp, _vp, _vp],
        "cpfit_spd_inverse_rows": [_int, _int, _i64, _vp, _i64, ctypes.c_double, _vp,
                                   ctypes.POINTER(_i64), _vp],
        "cpfit_batched_symv": [_int, _int, _i64, _vp, _vp, _vp, _vp],
        "cpfit_check_finite": [_int, _i64, _vp, _vp, _vp],
        "cpfit_tttp_loss": [_vp, _int, _int, _vp, _PP, _int, _vp, _vp, ctypes.POINTER(_i64),
                            _vp],
        "cpfit_loss_eval": [_int, _int, _i64, _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(_i64),
                            _vp],
        "cpfit_ccd_gen_weights": [_vp, _int, _int, _PP, _vp, _vp, _vp, _vp, _vp,
                                  ctypes.POINTER(_i64), _vp],
        "cpfit_ccd_gen_update": [_i64, _vp, _vp, ctypes.c_double, _vp, _vp, _vp],
        "cpfit_ccd_gen_model": [_vp, _int, _vp, _vp, _vp, _vp],
        "cpfit_from_coords": [_int, ctypes.POINTER(_i64), _i64, _int, _PP, _vp, _vp, _vp,
                              ctypes.POINTER(_i64), ctypes.POINTER(_int), _vp],
        "cpfit_ccd_fold": [_vp, _int, _PP, _PP, _vp, _vp],
        "cpfit_ccd_finalize": [_i64, _vp, ctypes.c_double, _vp, _vp],
        "cpfit_probe_gather": [_vp, _int, _int, _PP, _i64, _vp, _i64, _vp],
        "cpfit_probe_l2_read": [_vp, _i64, _int, _vp, _i64, _vp],
        "cpfit_solve_rows": [_int, _int, _i64, _vp, _i64, _vp, ctypes.c_double, _vp,
                             ctypes.POINTER(_i64), _vp],
        "cpfit_dense_reduce": [_int, _i64, _i64, _int, _vp, _vp, _int, _vp, _vp],
        "cpfit_khatri_rao": [_int, _i64, _i64, _int, _vp, _vp, _vp, _vp],
        "cpfit_dense_mttkrp": [_int, _i64, _i64, _i64, _int, _vp, _vp, _vp, _vp, _int, _vp,
                               _vp],
        "cpfit_dense_xc": [_int, _i64, _i64, _i64, _int, _vp, _vp, _vp, _vp],
        "cpfit_dense_gram": [_int, _int, ctypes.POINTER(_i64), _int, _PP, _vp, _vp],
        "cpfit_als_update": [_vp, _int, _int, _int, _vp, _int, _PP, ctypes.c_double, _vp, _vp,
                             _vp, ctypes.POINTER(_i64), _vp],
        "cpfit_gram_matvec": [_vp, _int, _int, _int, _vp, _int, _PP, _vp, _vp, _vp, _vp],
        "cpfit_cg_rows_init": [_int, _i64, _int, ctypes.c_double, ctypes.c_double, _vp, _vp,
                               _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
        "cpfit_cg_rows_step": [_int, _i64, _int, ctypes.c_double, _vp, _vp, _vp, _vp, _vp, _vp,
                               _vp, _vp, _vp],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = _int
    _lib = L
    return L


def last_error() -> str:
    return load().cpfit_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    """Map a C-ABI status onto the reference's exception types."""
    if status == OK:
        return
    msg = last_error()
    if status in (EINVAL, ENEGWEIGHT):
        raise ValueError(msg)
    if status in (ESINGULAR, EEMPTYROW):
        raise NumericalError(msg)
    if status == ENONFINITE:
        raise NumericalError(msg)
    if status == ENOMEM:
        raise MemoryError(msg)
    raise CpfitError(f"{what}: {msg}" if what else msg)


def ptr_array(ptrs) -> ctypes.Array:
    arr = (ctypes.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr

"""ctypes binding of libpolyjac_b200.so — the C ABI declared in include/polyjac_b200.h.

The product path has no fallback: if the shared library is missing or cannot be loaded,
every call raises. Build it with `python -m paper_1201_0499_b200.build` (or
`__graft_entry__.build()`); it is built in-tree so it ships with the repo snapshot.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("PJ_LIB_PATH") or os.path.join(HERE, "libpolyjac_b200.so")  # override: experiments

PJ_OK, PJ_EINVAL, PJ_ERANGE, PJ_ECUDA, PJ_ENOMEM, PJ_ENONFINITE, PJ_EFORMAT = 0, 1, 2, 3, 4, 5, 6
PJ_PREC_D, PJ_PREC_DD = 1, 2
PJ_ORDER_REF, PJ_ORDER_FAST = 0x10, 0x20
PJ_OP_NEWTON = 0x100
PJ_NEWTON_MIXED = 0x400
PJ_VALIDATE = 0x200
PJ_CTX_WIDE = 0x1

EXPORTS = [
    "pj_last_error", "pj_version", "pj_validate", "pj_ctx_create", "pj_ctx_destroy", "pj_evaluate",
    "pj_evaluate_host", "pj_nonfinite_seen", "pj_layout_info", "pj_mons_slot", "pj_slot_targets",
    "pj_zero_mask", "pj_mult_counts", "pj_random_system", "pj_random_points", "pj_set_launch",
    "pj_get_launch", "pj_fp64_peak_probe", "pj_random_points_range", "pj_set_kernel_variant",
    "pj_system_read_file", "pj_system_read_text", "pj_system_view", "pj_system_free", "pj_system_write_file",
    "pj_system_write_text", "pj_newton_solve", "pj_newton_step", "pj_newton_host",
    "pj_ctx_create_ex", "pj_layout_export", "pj_structural_zeros", "pj_debug_corrupt_coeff",
    "pj_fp64_pipe_probe", "pj_validate_ragged", "pj_ctx_create_ragged", "pj_random_ragged_system",
]


class SystemDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("m", ctypes.c_int32), ("k", ctypes.c_int32), ("d", ctypes.c_int32),
                ("positions", ctypes.c_void_p), ("exponents", ctypes.c_void_p), ("coeffs", ctypes.c_void_p)]


class RaggedDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("d", ctypes.c_int32), ("row_off", ctypes.c_void_p),
                ("term_off", ctypes.c_void_p), ("positions", ctypes.c_void_p), ("exponents", ctypes.c_void_p),
                ("coeffs", ctypes.c_void_p)]


class PolyjacError(RuntimeError):
    """CUDA / internal failure of the native library (PJ_ECUDA, PJ_ENOMEM)."""


class FormatError(RuntimeError):
    """Malformed system file (PJ_EFORMAT): polyjac::FormatError, ref include/polyjac/io.hpp:19-21."""


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise ImportError(f"{SO_PATH} is missing: build it with `python -m paper_1201_0499_b200.build` "
                          "(no CPU fallback exists)")
    L = ctypes.CDLL(SO_PATH)
    vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    i32p, i64p = ctypes.POINTER(i32), ctypes.POINTER(i64)
    L.pj_last_error.restype = ctypes.c_char_p
    L.pj_version.restype = ctypes.c_char_p
    L.pj_validate.argtypes = [ctypes.POINTER(SystemDesc), ctypes.c_char_p, ctypes.c_size_t]
    L.pj_ctx_create.argtypes = [ctypes.POINTER(SystemDesc), ctypes.c_int, ctypes.POINTER(vp)]
    L.pj_ctx_create_ex.argtypes = [ctypes.POINTER(SystemDesc), ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    L.pj_ctx_destroy.argtypes = [vp]
    L.pj_ctx_destroy.restype = None
    L.pj_evaluate.argtypes = [vp, ctypes.c_int, vp, i64, vp, vp]
    L.pj_evaluate_host.argtypes = [vp, ctypes.c_int, vp, i64, vp]
    L.pj_nonfinite_seen.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_int)]
    L.pj_layout_info.argtypes = [vp, i32p, i32p, i32p, i32p, i64p]
    L.pj_mons_slot.argtypes = [i64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, i64p]
    L.pj_slot_targets.argtypes = [vp, i64, vp]
    L.pj_zero_mask.argtypes = [vp, vp, i64]
    L.pj_zero_mask.restype = i64
    L.pj_mult_counts.argtypes = [vp, i64, vp]
    L.pj_random_system.argtypes = [ctypes.c_int] * 4 + [u64, vp, vp, vp]
    L.pj_random_points.argtypes = [ctypes.c_int, i64, u64, vp]
    L.pj_random_points_range.argtypes = [ctypes.c_int, i64, i64, u64, vp]
    L.pj_set_launch.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    L.pj_get_launch.argtypes = [vp, ctypes.c_int, i32p, i32p, i32p, i64p, i32p]
    L.pj_set_kernel_variant.argtypes = [vp, ctypes.c_int, ctypes.c_int]
    L.pj_system_read_file.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp)]
    L.pj_system_read_text.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(vp)]
    L.pj_system_view.argtypes = [vp, ctypes.POINTER(SystemDesc)]
    L.pj_system_free.argtypes = [vp]
    L.pj_system_free.restype = None
    L.pj_system_write_file.argtypes = [ctypes.POINTER(SystemDesc), ctypes.c_char_p]
    L.pj_system_write_text.argtypes = [ctypes.POINTER(SystemDesc), ctypes.c_char_p, i64]
    L.pj_system_write_text.restype = i64
    L.pj_newton_solve.argtypes = [vp, ctypes.c_int, vp, vp, vp, i64, vp, vp, vp, vp]
    L.pj_newton_step.argtypes = [vp, ctypes.c_int, vp, vp, i64, vp, vp, vp, vp, vp]
    L.pj_newton_host.argtypes = [vp, ctypes.c_int, vp, vp, i64, ctypes.c_int, vp, vp, vp]
    L.pj_fp64_peak_probe.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    L.pj_fp64_pipe_probe.argtypes = [ctypes.c_int, vp]
    L.pj_layout_export.argtypes = [vp, vp, vp, vp]
    L.pj_structural_zeros.argtypes = [vp, vp]
    L.pj_structural_zeros.restype = i64
    L.pj_debug_corrupt_coeff.argtypes = [vp, i64, ctypes.c_double]
    L.pj_validate_ragged.argtypes = [ctypes.POINTER(RaggedDesc), ctypes.c_char_p, ctypes.c_size_t]
    L.pj_ctx_create_ragged.argtypes = [ctypes.POINTER(RaggedDesc), ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp)]
    L.pj_random_ragged_system.argtypes = [ctypes.c_int] * 6 + [u64, i64p, i64p, vp, vp, vp, vp, vp]
    for name in EXPORTS:
        getattr(L, name)  # fail loudly on a stale library
    _lib = L
    return L


def last_error() -> str:
    return lib().pj_last_error().decode()


def check(rc: int, what: str = "") -> None:
    """Map a status code onto the exception the reference throws for the same condition."""
    if rc == PJ_OK:
        return
    msg = last_error() or what
    if rc in (PJ_EINVAL, PJ_ENONFINITE):
        raise ValueError(msg)          # std::invalid_argument
    if rc == PJ_ERANGE:
        raise IndexError(msg)          # std::out_of_range
    if rc == PJ_ENOMEM:
        raise MemoryError(msg)
    if rc == PJ_EFORMAT:
        raise FormatError(msg)
    raise PolyjacError(msg)

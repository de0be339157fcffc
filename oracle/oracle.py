"""ORACLE — test infrastructure only.

ctypes bindings for the CPU restatement (oracle/_build/liboracle.so, built from
oracle/oracle.cpp) and, when present, the unmodified reference library compiled from
/root/reference/proj/src (oracle/_ref/libpolyjac_ref.so, built by oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
import this module; the product package (paper_1201_0499_b200/) never does.

Array conventions (shared with the product's C ABI, include/polyjac_b200.h):
  pos, exps  int32 [n*m*k]          S_m order, s = p*m + g, slot s*k + j (ref system.hpp:28-31)
  coeffs     float64 [n*m, 4]       (re_hi, re_lo, im_hi, im_lo)
  points     float64 [B, n, W]      W = 2 (complex double) or 4 (complex double-double)
  out        float64 [B, n+n*n, W]  values[n] then the row-major Jacobian (ref system.hpp:48-54)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libpolyjac_ref.so")
DROPIN_BIN = os.path.join(HERE, "_ref", "test_dropin")
# the reference's own doctest suites, built unmodified (oracle/shim/doctest.h, oracle/Makefile)
REF_SUITES = ["test_system", "test_packing", "test_kernels", "test_oracle", "test_engine", "test_io"]
DROPIN_ENGINE_BIN = os.path.join(HERE, "_ref", "test_engine_b200")
REF_CLI_SUITE = os.path.join(HERE, "_ref", "test_cli")
REF_SRC = "/root/reference/proj"

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


def build(ref: bool | None = None) -> None:
    """Compile the oracle (always) and oracle/_ref (when the reference sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "-j8", "ref", "refsuites"], check=True)
        # the C++ drop-in checks link the product library; build them only once that exists
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_1201_0499_b200", "libpolyjac_b200.so")):
            subprocess.run(["make", "-s", "-C", HERE, "-j8", "dropin", "dropin-engine"], check=True)


_oracle = None
_ref = None


def lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = ctypes.CDLL(ORACLE_SO)
        L.oracle_evaluate.argtypes = [ctypes.c_int] * 5 + [_i32p, _i32p, _f64p, _f64p, ctypes.c_long,
                                                           _f64p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_evaluate.restype = ctypes.c_int
        L.oracle_evaluate_ragged.argtypes = [ctypes.c_int] * 3 + [_i32p] * 4 + [_f64p, _f64p, ctypes.c_long, _f64p,
                                                                        ctypes.c_void_p, ctypes.c_int]
        L.oracle_evaluate_ragged.restype = ctypes.c_int
        L.oracle_speelpenning.argtypes = [ctypes.c_int, ctypes.c_int, _f64p, _f64p,
                                          ctypes.POINTER(ctypes.c_ulonglong)]
        L.oracle_cdd_mul.argtypes = [_f64p, _f64p, _f64p]
        L.oracle_cdd_add.argtypes = [_f64p, _f64p, _f64p]
        L.oracle_mons_slot.argtypes = [ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.oracle_mons_slot.restype = ctypes.c_longlong
        L.oracle_zero_mask.argtypes = [ctypes.c_int] * 3 + [_i32p, _i64p]
        L.oracle_zero_mask.restype = ctypes.c_longlong
        L.oracle_newton_solve.argtypes = [ctypes.c_int, ctypes.c_int, _f64p, _f64p, ctypes.c_void_p, ctypes.c_long,
                                          _f64p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        L.oracle_newton_solve.restype = ctypes.c_int
        _oracle = L
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        L = ctypes.CDLL(REF_SO)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_random_system.argtypes = [ctypes.c_int] * 4 + [ctypes.c_ulonglong, _i32p, _i32p, _f64p]
        L.ref_random_points.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong, _f64p]
        L.ref_validate.argtypes = [ctypes.c_int] * 4 + [_i32p, _i32p, _f64p, ctypes.c_longlong]
        L.ref_build_layout.argtypes = [ctypes.c_int] * 4 + [_i32p, _i32p, _f64p,
                                                            np.ctypeslib.ndpointer(np.uint8), np.ctypeslib.ndpointer(np.uint8), _f64p]
        L.ref_mons_slot.argtypes = [ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.ref_mons_slot.restype = ctypes.c_longlong
        L.ref_zero_mask.argtypes = [ctypes.c_int] * 4 + [_i32p, _i32p, _f64p, _i64p]
        L.ref_zero_mask.restype = ctypes.c_longlong
        L.ref_slot_targets.argtypes = [ctypes.c_int] * 4 + [_i32p, _i32p, _f64p, _i64p]
        L.ref_evaluate.argtypes = [ctypes.c_int] * 4 + [_i32p, _i32p, _f64p, _f64p, ctypes.c_longlong, _f64p,
                                                        ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                        ctypes.POINTER(ctypes.c_ulonglong), ctypes.POINTER(ctypes.c_double)]
        L.ref_naive.argtypes = [ctypes.c_int] * 4 + [_i32p, _i32p, _f64p, _f64p, _f64p]
        L.ref_write_system.argtypes = [ctypes.c_int] * 4 + [_i32p, _i32p, _f64p, ctypes.c_char_p, ctypes.c_longlong]
        L.ref_write_system.restype = ctypes.c_longlong
        L.ref_read_system.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong]
        _ref = L
    return _ref


class RefError(RuntimeError):
    pass


def _ref_err():
    return RefError(ref().ref_last_error().decode())


# --------------------------------------------------------------------------- oracle calls
def evaluate(prec, sysd, points, threads=1, magsum=False, counts=False):
    """CPU restatement of EvaluationContext::evaluate over a batch (see module doc).

    prec: "d" (complex double, reference arithmetic) or "dd" (complex double-double).
    sysd: dict with n, m, k, d, pos, exps, coeffs. Returns out (and magsum / counts)."""
    n, m, k, d = sysd["n"], sysd["m"], sysd["k"], sysd["d"]
    W = 2 if prec == "d" else 4
    pts = np.ascontiguousarray(points, dtype=np.float64)
    B = pts.shape[0]
    assert pts.shape == (B, n, W), pts.shape
    out = np.empty((B, n + n * n, W), np.float64)
    ms = np.empty((B, n + n * n), np.float64) if magsum else None
    cnt = (ctypes.c_ulonglong * 5)() if counts else None
    rc = lib().oracle_evaluate(1 if prec == "d" else 2, n, m, k, d, sysd["pos"], sysd["exps"], sysd["coeffs"],
                               pts, B, out, ms.ctypes.data if ms is not None else None,
                               ctypes.addressof(cnt) if cnt is not None else None, threads)
    if rc:
        raise RuntimeError("oracle_evaluate failed")
    res = [out]
    if magsum:
        res.append(ms)
    if counts:
        res.append(dict(zip(["powers", "factors", "stage2", "speelpenning", "stage3"], list(cnt))))
    return res[0] if len(res) == 1 else tuple(res)


def evaluate_ragged(prec, rsys, points, threads=1, magsum=False):
    """Ragged restatement (oracle.cpp: evaluate_one_ragged). rsys: dict with n, d, row_off [n+1],
    term_off [T+1], pos, exps [term_off[T]], coeffs [T, 4]."""
    n, d = rsys["n"], rsys["d"]
    W = 2 if prec == "d" else 4
    pts = np.ascontiguousarray(points, dtype=np.float64)
    B = pts.shape[0]
    assert pts.shape == (B, n, W), pts.shape
    out = np.empty((B, n + n * n, W), np.float64)
    ms = np.empty((B, n + n * n), np.float64) if magsum else None
    arr = [np.ascontiguousarray(rsys[key], np.int32) for key in ("row_off", "term_off", "pos", "exps")]
    rc = lib().oracle_evaluate_ragged(1 if prec == "d" else 2, n, d, *arr,
                                      np.ascontiguousarray(rsys["coeffs"], np.float64).reshape(-1), pts, B, out,
                                      ms.ctypes.data if ms is not None else None, threads)
    if rc:
        raise RuntimeError("oracle_evaluate_ragged failed")
    return (out, ms) if magsum else out


def newton_solve(prec, n, evals, points, target=None, threads=1):
    """CPU restatement of the Newton corrector (paper_1201_0499_b200/csrc/newton.cu): per point
    solve J dx = y - f from the evaluator's output and return (x + dx, norms [B, 2], status [B]).
    prec: "d", "dd", or "mixed" (dd input; complex-double factors + dd iterative refinement)."""
    W = 2 if prec == "d" else 4
    ev = np.ascontiguousarray(evals, np.float64)
    pts = np.ascontiguousarray(points, np.float64)
    B = pts.shape[0]
    assert pts.shape == (B, n, W) and ev.shape == (B, n + n * n, W), (pts.shape, ev.shape)
    tg = None
    if target is not None:
        tg = np.ascontiguousarray(target, np.float64)
        assert tg.shape == pts.shape
    out = np.empty_like(pts)
    norms = np.empty((B, 2), np.float64)
    status = np.empty(B, np.int32)
    rc = lib().oracle_newton_solve({"d": 1, "dd": 2, "mixed": 3}[prec], n, ev, pts, tg.ctypes.data if tg is not None else None,
                                   B, out, norms.ctypes.data, status.ctypes.data, threads)
    if rc:
        raise RuntimeError("oracle_newton_solve failed")
    return out, norms, status


def speelpenning(prec, vals):
    vals = np.ascontiguousarray(vals, np.float64)
    k = vals.shape[0]
    L = np.zeros((k, vals.shape[1]), np.float64)
    mults = ctypes.c_ulonglong(0)
    lib().oracle_speelpenning(1 if prec == "d" else 2, k, vals, L, ctypes.byref(mults))
    return L, mults.value


def cdd_mul(a, b):
    r = np.zeros(4)
    lib().oracle_cdd_mul(np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64), r)
    return r


def cdd_add(a, b):
    r = np.zeros(4)
    lib().oracle_cdd_add(np.ascontiguousarray(a, np.float64), np.ascontiguousarray(b, np.float64), r)
    return r


def mons_slot(s, kind, var, n, m):
    return lib().oracle_mons_slot(s, 0 if kind == "value" else 1, var, n, m)


def zero_mask(sysd):
    n, m, k = sysd["n"], sysd["m"], sysd["k"]
    buf = np.empty((n * n + n) * m, np.int64)
    ln = lib().oracle_zero_mask(n, m, k, sysd["pos"], buf)
    return buf[:ln].copy()


# --------------------------------------------------------------------------- reference calls
def ref_random_system(n, m, k, d, seed):
    nm = n * m
    pos = np.empty(nm * k, np.int32)
    exps = np.empty(nm * k, np.int32)
    coeffs = np.empty((nm, 4), np.float64)
    if ref().ref_random_system(n, m, k, d, seed, pos, exps, coeffs):
        raise _ref_err()
    return dict(n=n, m=m, k=k, d=d, pos=pos, exps=exps, coeffs=coeffs)


def ref_random_points(n, count, seed):
    out = np.empty((count, n, 2), np.float64)
    if ref().ref_random_points(n, count, seed, out):
        raise _ref_err()
    return out


def ref_evaluate(sysd, points, threads=1, block_size=32, workers=1, timing=False):
    n = sysd["n"]
    pts = np.ascontiguousarray(points, np.float64)
    B = pts.shape[0]
    out = np.empty((B, n + n * n, 2), np.float64)
    mults = ctypes.c_ulonglong(0)
    secs = ctypes.c_double(0)
    if ref().ref_evaluate(n, sysd["m"], sysd["k"], sysd["d"], sysd["pos"], sysd["exps"], sysd["coeffs"],
                          pts, B, out, threads, block_size, workers, ctypes.byref(mults), ctypes.byref(secs)):
        raise _ref_err()
    if timing:
        return out, mults.value, secs.value
    return out


def ref_naive(sysd, point):
    n = sysd["n"]
    out = np.empty((n + n * n, 2), np.float64)
    if ref().ref_naive(n, sysd["m"], sysd["k"], sysd["d"], sysd["pos"], sysd["exps"], sysd["coeffs"],
                       np.ascontiguousarray(point, np.float64), out):
        raise _ref_err()
    return out


def ref_zero_mask(sysd):
    n, m = sysd["n"], sysd["m"]
    buf = np.empty((n * n + n) * m, np.int64)
    ln = ref().ref_zero_mask(n, m, sysd["k"], sysd["d"], sysd["pos"], sysd["exps"], sysd["coeffs"], buf)
    return buf[:ln].copy()


def ref_slot_targets(sysd):
    n, m, k = sysd["n"], sysd["m"], sysd["k"]
    buf = np.empty((n * m, k + 1), np.int64)
    if ref().ref_slot_targets(n, m, k, sysd["d"], sysd["pos"], sysd["exps"], sysd["coeffs"], buf):
        raise _ref_err()
    return buf


def ref_validate(sysd, nterms=None):
    n, m = sysd["n"], sysd["m"]
    if nterms is None:
        nterms = n * m
    nv = ref().ref_validate(n, m, sysd["k"], sysd["d"], sysd["pos"], sysd["exps"], sysd["coeffs"], nterms)
    return nv, ref().ref_last_error().decode()


def ref_mons_slot(s, kind, var, n, m):
    return ref().ref_mons_slot(s, 0 if kind == "value" else 1, var, n, m)


def ref_write_system(sysd):
    n, m, k, d = sysd["n"], sysd["m"], sysd["k"], sysd["d"]
    ln = ref().ref_write_system(n, m, k, d, sysd["pos"], sysd["exps"], sysd["coeffs"], None, 0)
    buf = ctypes.create_string_buffer(ln + 1)
    ref().ref_write_system(n, m, k, d, sysd["pos"], sysd["exps"], sysd["coeffs"], buf, ln + 1)
    return buf.value.decode()


def ref_read_system(text):
    """Reference read_system on a string; raises RefError (FormatError text) on bad input."""
    dims = (ctypes.c_int * 4)()
    if ref().ref_read_system(text.encode(), dims, None, None, None, 0):
        raise _ref_err()
    n, m, k, d = list(dims)
    pos = np.empty(n * m * k, np.int32)
    exps = np.empty(n * m * k, np.int32)
    coeffs = np.empty((n * m, 4), np.float64)
    ref().ref_read_system(text.encode(), dims, pos.ctypes.data, exps.ctypes.data, coeffs.ctypes.data, n * m)
    return dict(n=n, m=m, k=k, d=d, pos=pos, exps=exps, coeffs=coeffs)

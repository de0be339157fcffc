"""Host-side mirror of the reference's C++ API for the hot path, over the C ABI.

Reference surface (ref = /root/reference/proj):
  PolynomialSystem / Term / MonomialSupport   ref include/polyjac/system.hpp:14-42
  validate_system                             ref src/system.cpp:21-64
  random_system / random_points / random_point ref src/system.cpp:66-118
  GridConfig                                  ref include/polyjac/engine.hpp:16-19
  EvaluationContext(sys, grid)                ref src/engine.cpp:168-179
    .evaluate(point) -> EvaluationResult      ref src/engine.cpp:181-230
    .evaluate_batch(points, repeat)           ref src/engine.cpp:232-260
    .mults() / .masked_slots_clean()          ref include/polyjac/engine.hpp:104-108
  mons_slot / zero_mask / stage2_slot_targets ref src/packing.cpp:8-72, src/kernels.cpp:129-137

Same names, argument meaning and error behaviour (ValueError where the reference throws
std::invalid_argument, IndexError for std::out_of_range). Additions for the B200 path:
complex double-double evaluation (`evaluate_dd`, `precision="dd"`) and batched device-tensor
evaluation (`evaluate_device`) on a CUDA stream. All arithmetic runs in the CUDA kernels of
libpolyjac_b200.so; nothing here computes results on the CPU.
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from typing import List, Sequence

import numpy as np

from . import _lib
from ._lib import PJ_ORDER_FAST, PJ_ORDER_REF, PJ_PREC_D, PJ_PREC_DD, RaggedDesc, SystemDesc, check, lib


# --------------------------------------------------------------------------- system model
@dataclass
class MonomialSupport:
    positions: List[int]
    exponents: List[int]

    def size(self) -> int:
        return len(self.positions)


@dataclass
class Term:
    coeff: complex
    support: MonomialSupport


@dataclass
class PolynomialSystem:
    """n polynomials in n variables, m monomials each, k variables per monomial, degrees in
    [1, d]; terms flat in S_m order (monomial g of polynomial p at p*m + g).

    Stored as arrays: positions/exponents int32 [n*m, k]; coeffs float64 [n*m, 4] =
    (re_hi, re_lo, im_hi, im_lo) so double-double coefficients are representable."""
    n: int
    m: int
    k: int
    d: int
    positions: np.ndarray
    exponents: np.ndarray
    coeffs: np.ndarray

    @staticmethod
    def from_terms(n: int, m: int, k: int, d: int, terms: Sequence[Term]) -> "PolynomialSystem":
        nt = len(terms)
        kk = max(k, 0)
        pos = np.full((nt, kk), -1, np.int32)
        exps = np.zeros((nt, kk), np.int32)
        co = np.zeros((nt, 4), np.float64)
        bad = False
        for s, t in enumerate(terms):
            if len(t.support.positions) != k or len(t.support.exponents) != k:
                bad = True
                continue
            pos[s] = t.support.positions
            exps[s] = t.support.exponents
            c = complex(t.coeff)
            co[s] = (c.real, 0.0, c.imag, 0.0)
        sys = PolynomialSystem(n, m, k, d, pos, exps, co)
        sys._shape_error = bad or nt != n * m
        return sys

    def monomial_count(self) -> int:
        return self.n * self.m

    def term(self, p: int, g: int) -> Term:
        s = p * self.m + g
        c = self.coeffs[s]
        return Term(complex(c[0] + c[1], c[2] + c[3]),
                    MonomialSupport([int(v) for v in self.positions[s]], [int(v) for v in self.exponents[s]]))

    @property
    def terms(self) -> List[Term]:
        return [self.term(s // self.m, s % self.m) for s in range(self.n * self.m)]

    def _desc(self):
        pos = np.ascontiguousarray(self.positions, np.int32).reshape(-1)
        exps = np.ascontiguousarray(self.exponents, np.int32).reshape(-1)
        co = np.ascontiguousarray(self.coeffs, np.float64).reshape(-1)
        keep = (pos, exps, co)
        desc = SystemDesc(self.n, self.m, self.k, self.d, pos.ctypes.data, exps.ctypes.data, co.ctypes.data)
        if getattr(self, "_shape_error", False) or pos.size != self.n * self.m * max(self.k, 0):
            desc.positions = desc.exponents = desc.coeffs = None  # "term count is not n*m"
        return desc, keep


@dataclass
class Violation:
    poly: int
    mono: int
    rule: str

    def describe(self) -> str:
        return self.rule


@dataclass
class ValidationReport:
    violations: List[Violation] = field(default_factory=list)

    def ok(self) -> bool:
        return not self.violations


def validate_system(sys: PolynomialSystem) -> ValidationReport:
    desc, keep = sys._desc()
    buf = ctypes.create_string_buffer(512)
    nv = lib().pj_validate(ctypes.byref(desc), buf, 512)
    rep = ValidationReport()
    if nv > 0:
        rep.violations.append(Violation(-1, -1, buf.value.decode()))
        rep.violations.extend(Violation(-1, -1, "") for _ in range(nv - 1))
    return rep


def random_system(n: int, m: int, k: int, d: int, seed: int) -> PolynomialSystem:
    """Bit-identical to the reference generator (ref src/system.cpp:66-101)."""
    nm = max(n, 0) * max(m, 0)
    pos = np.empty((nm, max(k, 1)), np.int32)
    exps = np.empty((nm, max(k, 1)), np.int32)
    co = np.empty((nm, 4), np.float64)
    check(lib().pj_random_system(n, m, k, d, seed, pos.ctypes.data, exps.ctypes.data, co.ctypes.data))
    return PolynomialSystem(n, m, k, d, pos, exps, co)


# --------------------------------------------------------------------------- ragged systems (f4)
@dataclass
class RaggedSystem:
    """Non-uniform m and k (include/polyjac_b200.h pj_ragged_desc): polynomial p
    owns terms [row_off[p], row_off[p+1]), term t owns positions/exponents [term_off[t],
    term_off[t+1]); coeffs float64 [T, 4] = (re_hi, re_lo, im_hi, im_lo). Per-term rules as
    validate_system (ref src/system.cpp:21-64)."""
    n: int
    d: int
    row_off: np.ndarray
    term_off: np.ndarray
    positions: np.ndarray
    exponents: np.ndarray
    coeffs: np.ndarray

    @property
    def term_count(self) -> int:
        return int(self.row_off[self.n])

    def m_of(self, p: int) -> int:
        return int(self.row_off[p + 1] - self.row_off[p])

    def k_of(self, t: int) -> int:
        return int(self.term_off[t + 1] - self.term_off[t])

    def term(self, p: int, g: int) -> Term:
        t = int(self.row_off[p]) + g
        a, b = int(self.term_off[t]), int(self.term_off[t + 1])
        c = self.coeffs[t]
        return Term(complex(c[0] + c[1], c[2] + c[3]),
                    MonomialSupport([int(v) for v in self.positions[a:b]], [int(v) for v in self.exponents[a:b]]))

    @staticmethod
    def from_uniform(sys: PolynomialSystem) -> "RaggedSystem":
        """The same uniform system in ragged form (evaluates bit-identically)."""
        nm = sys.n * sys.m
        return RaggedSystem(sys.n, sys.d, np.arange(sys.n + 1, dtype=np.int32) * sys.m,
                            np.arange(nm + 1, dtype=np.int32) * sys.k,
                            np.ascontiguousarray(sys.positions, np.int32).reshape(-1).copy(),
                            np.ascontiguousarray(sys.exponents, np.int32).reshape(-1).copy(),
                            np.ascontiguousarray(sys.coeffs, np.float64).reshape(nm, 4).copy())

    @staticmethod
    def from_polynomials(n: int, d: int, polys: Sequence[Sequence[Term]]) -> "RaggedSystem":
        """From n lists of Terms (each term with its own support size)."""
        ro, to, ps, es, cs = [0], [0], [], [], []
        for terms in polys:
            for t in terms:
                ps.extend(t.support.positions)
                es.extend(t.support.exponents)
                to.append(to[-1] + len(t.support.positions))
                c = complex(t.coeff)
                cs.append((c.real, 0.0, c.imag, 0.0))
            ro.append(ro[-1] + len(terms))
        return RaggedSystem(n, d, np.array(ro, np.int32), np.array(to, np.int32), np.array(ps, np.int32),
                            np.array(es, np.int32), np.array(cs, np.float64).reshape(-1, 4))

    def as_dict(self) -> dict:
        """Array dict for the oracle (tests only)."""
        return dict(n=self.n, d=self.d, row_off=self.row_off, term_off=self.term_off, pos=self.positions,
                    exps=self.exponents, coeffs=self.coeffs)

    def _desc(self):
        arrs = (np.ascontiguousarray(self.row_off, np.int32), np.ascontiguousarray(self.term_off, np.int32),
                np.ascontiguousarray(self.positions, np.int32), np.ascontiguousarray(self.exponents, np.int32),
                np.ascontiguousarray(self.coeffs, np.float64))
        if arrs[0].size != self.n + 1 or arrs[1].size < 1:
            raise ValueError("ragged system: row_off needs n + 1 entries and term_off at least one")
        T = int(arrs[0][-1])
        if arrs[1].size != T + 1 or arrs[2].size < int(arrs[1][-1]) or arrs[3].size < int(arrs[1][-1]) \
                or arrs[4].size != 4 * T:
            raise ValueError("ragged system: array sizes do not match row_off / term_off")
        desc = RaggedDesc(self.n, self.d, *(a.ctypes.data for a in arrs))
        return desc, arrs


def validate_ragged_system(sys: RaggedSystem) -> ValidationReport:
    desc, keep = sys._desc()
    buf = ctypes.create_string_buffer(512)
    nv = lib().pj_validate_ragged(ctypes.byref(desc), buf, 512)
    rep = ValidationReport()
    if nv > 0:
        rep.violations.append(Violation(-1, -1, buf.value.decode()))
        rep.violations.extend(Violation(-1, -1, "") for _ in range(nv - 1))
    return rep


def random_ragged_system(n: int, m_range, k_range, d: int, seed: int) -> RaggedSystem:
    """m_p uniform in m_range = (lo, hi) per polynomial, k_t uniform in k_range per term, then the
    reference generator's per-term draws (pj_random_ragged_system)."""
    T, S = ctypes.c_int64(), ctypes.c_int64()
    L = lib()
    args = (n, int(m_range[0]), int(m_range[1]), int(k_range[0]), int(k_range[1]), d, seed)
    check(L.pj_random_ragged_system(*args, ctypes.byref(T), ctypes.byref(S), None, None, None, None, None))
    ro = np.empty(n + 1, np.int32)
    to = np.empty(T.value + 1, np.int32)
    ps = np.empty(max(S.value, 1), np.int32)
    es = np.empty(max(S.value, 1), np.int32)
    co = np.empty((T.value, 4), np.float64)
    check(L.pj_random_ragged_system(*args, None, None, ro.ctypes.data, to.ctypes.data, ps.ctypes.data,
                                    es.ctypes.data, co.ctypes.data))
    return RaggedSystem(n, d, ro, to, ps[:S.value], es[:S.value], co)


def random_points(n: int, count: int, seed: int) -> np.ndarray:
    """count points, complex128 [count, n], one seeded stream (ref src/system.cpp:103-114)."""
    out = np.empty((count, n, 2), np.float64)
    check(lib().pj_random_points(n, count, seed, out.ctypes.data))
    return out.view(np.complex128).reshape(count, n)


def random_point(n: int, seed: int) -> np.ndarray:
    return random_points(n, 1, seed)[0]


def to_dd(points) -> np.ndarray:
    """complex128 [..., n] -> double-double planes float64 [..., n, 4] with zero low words."""
    z = np.asarray(points, np.complex128)
    out = np.zeros(z.shape + (4,), np.float64)
    out[..., 0] = z.real
    out[..., 2] = z.imag
    return out


# --------------------------------------------------------------------------- system files
def _from_handle(h) -> PolynomialSystem:
    desc = SystemDesc()
    check(lib().pj_system_view(h, ctypes.byref(desc)))
    n, m, k = desc.n, desc.m, desc.k
    nm = n * m
    pos = np.ctypeslib.as_array(ctypes.cast(desc.positions, ctypes.POINTER(ctypes.c_int32)), (nm * k,)).copy()
    exps = np.ctypeslib.as_array(ctypes.cast(desc.exponents, ctypes.POINTER(ctypes.c_int32)), (nm * k,)).copy()
    co = np.ctypeslib.as_array(ctypes.cast(desc.coeffs, ctypes.POINTER(ctypes.c_double)), (nm * 4,)).copy()
    lib().pj_system_free(h)
    return PolynomialSystem(n, m, k, desc.d, pos.reshape(nm, k), exps.reshape(nm, k), co.reshape(nm, 4))


def read_system(path: str) -> PolynomialSystem:
    """ref src/io.cpp:115-119; FormatError ("path:line: what") on malformed input."""
    h = ctypes.c_void_p()
    check(lib().pj_system_read_file(path.encode(), ctypes.byref(h)))
    return _from_handle(h)


def read_system_text(text: str, name: str = "<stream>") -> PolynomialSystem:
    """ref src/io.cpp:38-98 on an in-memory text."""
    h = ctypes.c_void_p()
    check(lib().pj_system_read_text(text.encode(), name.encode(), ctypes.byref(h)))
    return _from_handle(h)


def write_system_text(sys: PolynomialSystem) -> str:
    """ref src/io.cpp:100-108: doubles with 17 significant digits, 1-based positions."""
    desc, keep = sys._desc()
    ln = lib().pj_system_write_text(ctypes.byref(desc), None, 0)
    if ln < 0:
        check(_lib.PJ_EINVAL)
    buf = ctypes.create_string_buffer(ln + 1)
    lib().pj_system_write_text(ctypes.byref(desc), buf, ln + 1)
    return buf.value.decode()


def write_system(sys: PolynomialSystem, path: str) -> None:
    desc, keep = sys._desc()
    check(lib().pj_system_write_file(ctypes.byref(desc), path.encode()))


def mons_slot(s: int, kind: str, var: int, n: int, m: int) -> int:
    """ref src/packing.cpp:8-17; IndexError where the reference throws std::out_of_range."""
    out = ctypes.c_int64(0)
    check(lib().pj_mons_slot(s, 0 if kind == "value" else 1, var, n, m, ctypes.byref(out)))
    return out.value


def mons_value_slot(s, n, m):
    return mons_slot(s, "value", -1, n, m)


def mons_deriv_slot(s, var, n, m):
    return mons_slot(s, "derivative", var, n, m)


# --------------------------------------------------------------------------- results
@dataclass
class GridConfig:
    block_size: int = 32
    workers: int = 0  # 0 = all hardware threads (the CPU pool's knob; the GPU grid ignores it)


@dataclass
class EvaluationResult:
    n: int
    values: np.ndarray    # complex128 [n]   (dd: float64 [n, 4])
    jacobian: np.ndarray  # complex128 [n*n] row-major by polynomial (dd: [n*n, 4])

    def jac(self, p: int, i: int):
        return self.jacobian[p * self.n + i]


@dataclass
class PackedLayout:
    """ref include/polyjac/packing.hpp:24-46: positions / exponents-minus-one bytes [n*m*k] in S_m
    order, coeffs complex128 [(k+1)*n*m] derivative-major (block j < k: a_j * c, block k: c)."""
    n: int
    m: int
    k: int
    d: int
    positions: np.ndarray
    exponents: np.ndarray
    coeffs: np.ndarray

    def monomial_count(self) -> int:
        return self.n * self.m

    def position(self, s: int, j: int) -> int:
        return int(self.positions[s * self.k + j])

    def exponent_minus_1(self, s: int, j: int) -> int:
        return int(self.exponents[s * self.k + j])

    def deriv_coeff(self, s: int, j: int) -> complex:
        return complex(self.coeffs[j * self.monomial_count() + s])

    def value_coeff(self, s: int) -> complex:
        return complex(self.coeffs[self.k * self.monomial_count() + s])

    def footprint_bytes(self) -> int:
        return int(self.positions.size + self.exponents.size)


@dataclass
class MultCounter:
    stage1_powers: int = 0
    stage1_factors: int = 0
    stage2: int = 0
    speelpenning: int = 0
    stage3: int = 0

    def total(self) -> int:
        return self.stage1_powers + self.stage1_factors + self.stage2 + self.stage3


@dataclass
class BatchReport:
    evals: int = 0
    wall_seconds: float = 0.0
    per_eval_seconds: float = 0.0
    mults: MultCounter = field(default_factory=MultCounter)


@dataclass
class BatchResult:
    results: List[EvaluationResult]
    report: BatchReport


def _flags(precision: str, order: str | None) -> int:
    if precision == "d":
        return PJ_PREC_D | (PJ_ORDER_FAST if order == "fast" else 0)
    if precision == "dd":
        return PJ_PREC_DD | (PJ_ORDER_REF if order == "ref" else 0)
    raise ValueError(f"unknown precision {precision!r} (expected 'd' or 'dd')")


def _nflags(precision: str, order: str | None) -> int:
    """Newton solves: 'd', 'dd', or 'mixed' (complex dd in and out, the Jacobian factored in complex
    double and refined with complex-dd residuals: PJ_NEWTON_MIXED, n <= 32)."""
    if precision == "mixed":
        return _flags("dd", order) | _lib.PJ_NEWTON_MIXED
    return _flags(precision, order)


class EvaluationContext:
    """Owns the packed system on one GPU (uploaded once) and evaluates points there.

    Like the reference, one context must not serve concurrent evaluate calls; use one per
    thread (or per device / stream)."""

    def __init__(self, sys: PolynomialSystem | RaggedSystem, grid: GridConfig | None = None, device: int = 0,
                 wide: bool = False):
        """wide=True lifts the reference's n <= 256 byte-encoding cap (pj_ctx_create_ex, PJ_CTX_WIDE).
        A RaggedSystem (non-uniform m / k) goes through pj_ctx_create_ragged;
        self.m / self.k are then the maxima."""
        grid = grid or GridConfig()
        if grid.block_size < 1:
            raise ValueError("block size must be >= 1")
        if grid.workers < 0:
            raise ValueError("workers must be >= 0")
        self.grid_ = GridConfig(grid.block_size, grid.workers if grid.workers > 0 else 1)
        self.device = device
        self.ragged = isinstance(sys, RaggedSystem)
        desc, keep = sys._desc()
        h = ctypes.c_void_p()
        opts = _lib.PJ_CTX_WIDE if wide else 0
        if self.ragged:
            check(lib().pj_ctx_create_ragged(ctypes.byref(desc), device, opts, ctypes.byref(h)))
        else:
            check(lib().pj_ctx_create_ex(ctypes.byref(desc), device, opts, ctypes.byref(h)))
        self._h = h
        if self.ragged:
            info = self.layout_info()
            self.n, self.m, self.k, self.d = info["n"], info["m"], info["k"], info["d"]
        else:
            self.n, self.m, self.k, self.d = sys.n, sys.m, sys.k, sys.d
        self._mults = MultCounter()
        self._clean = True
        self._zeros = None
        self._layout = None
        self._per_eval = None  # MultCounter of one evaluation (the tally is linear in the count)
        self._one_out = None   # staging array of the single-point API

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().pj_ctx_destroy(h)
            except Exception:
                pass
            self._h = None

    # ---- reference surface
    def grid(self) -> GridConfig:
        return self.grid_

    def mults(self) -> MultCounter:
        return self._mults

    def masked_slots_clean(self) -> bool:
        """True while every structural zero (Jacobian entry (p, i) with variable i in no monomial
        of polynomial p) of every result returned by evaluate / evaluate_batch / evaluate_dd has
        been an exact +0 in every word. The GPU path keeps no padded Mons buffer, so its masked
        slots (ref src/engine.cpp:262-269) are exactly these output entries."""
        return self._clean

    def _structural_zeros(self) -> np.ndarray:
        if self._zeros is None:
            mask = np.zeros(self.n * self.n, np.uint8)
            cnt = lib().pj_structural_zeros(self._h, mask.ctypes.data)
            if cnt < 0:
                check(_lib.PJ_EINVAL)
            self._zeros = self.n + np.nonzero(mask)[0]  # output rows of the [B, n + n*n, W] layout
        return self._zeros

    def _audit(self, out: np.ndarray) -> None:
        z = self._structural_zeros()
        if z.size and self._clean:
            self._clean = not np.any(out[:, z, :].view(np.uint64))

    def layout(self) -> "PackedLayout":
        """The reference's PackedLayout (ref include/polyjac/packing.hpp:24-46) of this context,
        bit-identical with build_layout (ref src/packing.cpp:19-52)."""
        if self._layout is None:
            nm, k = self.n * self.m, self.k
            pos = np.empty(nm * k, np.uint8)
            exps = np.empty(nm * k, np.uint8)
            co = np.empty(((k + 1) * nm, 2), np.float64)
            check(lib().pj_layout_export(self._h, pos.ctypes.data, exps.ctypes.data, co.ctypes.data))
            self._layout = PackedLayout(self.n, self.m, self.k, self.d, pos, exps, co.view(np.complex128).reshape(-1))
        return self._layout

    def layout_info(self):
        n, m, k, d = (ctypes.c_int32() for _ in range(4))
        fp = ctypes.c_int64()
        check(lib().pj_layout_info(self._h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(k), ctypes.byref(d),
                                   ctypes.byref(fp)))
        return dict(n=n.value, m=m.value, k=k.value, d=d.value, footprint_bytes=fp.value)

    def _tally(self, evals: int) -> MultCounter:
        c = (ctypes.c_uint64 * 5)()
        check(lib().pj_mult_counts(self._h, evals, ctypes.addressof(c)))
        return MultCounter(*[int(v) for v in c])

    def _add_tally(self, evals):
        # the closed-form counts are linear in the number of evaluations: one C call per context
        if self._per_eval is None:
            self._per_eval = self._tally(1)
        t = self._per_eval
        mc = self._mults
        if evals != 1:
            t = MultCounter(*[evals * getattr(t, f) for f in ("stage1_powers", "stage1_factors", "stage2",
                                                              "speelpenning", "stage3")])
        mc.stage1_powers += t.stage1_powers
        mc.stage1_factors += t.stage1_factors
        mc.stage2 += t.stage2
        mc.speelpenning += t.speelpenning
        mc.stage3 += t.stage3

    def evaluate_host(self, points: np.ndarray, precision: str = "d", order: str | None = None,
                      out: np.ndarray | None = None) -> np.ndarray:
        """Batched host-buffer evaluation. points: [B, n, W] float64 (W = 2 for 'd', 4 for 'dd');
        returns [B, n + n*n, W] (written into `out` when given — pass page-locked buffers, e.g.
        torch pin_memory() tensors' .numpy(), for full H2D/kernel/D2H overlap)."""
        W = 2 if precision == "d" else 4
        pts = np.ascontiguousarray(points, np.float64)
        if pts.ndim != 3 or pts.shape[1:] != (self.n, W):
            raise ValueError("evaluate: point dimension mismatch")
        B = pts.shape[0]
        shape = (B, self.n + self.n * self.n, W)
        if out is None:
            out = np.empty(shape, np.float64)
        elif out.shape != shape or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ValueError("evaluate: output buffer must be C-contiguous float64 of shape %s" % (shape,))
        check(lib().pj_evaluate_host(self._h, _flags(precision, order), pts.ctypes.data, B, out.ctypes.data))
        self._add_tally(B)
        return out

    def evaluate(self, point) -> EvaluationResult:
        """One point (sequence of n complex numbers) in complex double; bit-identical with the
        reference's EvaluationContext::evaluate."""
        z = np.ascontiguousarray(point, np.complex128).reshape(-1)
        if z.shape[0] != self.n:
            raise ValueError("evaluate: point dimension mismatch")
        pts = z.view(np.float64).reshape(1, self.n, 2)  # complex128 is (re, im) interleaved already
        if not np.isfinite(pts).all():
            raise ValueError("evaluate: non-finite coordinate")
        if self._one_out is None:  # results are copied out below: one staging array per context
            self._one_out = np.empty((1, self.n + self.n * self.n, 2), np.float64)
        out = self.evaluate_host(pts, "d", out=self._one_out)
        self._audit(out)
        c = out[0].view(np.complex128)[:, 0]
        return EvaluationResult(self.n, c[: self.n].copy(), c[self.n:].copy())

    def evaluate_dd(self, points_dd: np.ndarray, order: str | None = None) -> np.ndarray:
        """Complex double-double: points [B, n, 4] -> [B, n + n*n, 4]."""
        out = self.evaluate_host(points_dd, "dd", order)
        self._audit(out)
        return out

    def evaluate_batch(self, points, repeat: int) -> BatchResult:
        if repeat < 1:
            raise ValueError("evaluate_batch: repeat must be >= 1")
        pts = [np.asarray(p, np.complex128).reshape(-1) for p in points]
        for z in pts:
            if z.shape[0] != self.n:
                raise ValueError("evaluate: point dimension mismatch")
        before = MultCounter(**vars(self._mults))
        t0 = time.perf_counter()
        results = []
        if pts:
            arr = np.stack([np.stack([z.real, z.imag], -1) for z in pts])
            out = None
            for _ in range(repeat):
                out = self.evaluate_host(arr, "d")
                self._audit(out)
            c = out[..., 0] + 1j * out[..., 1]
            results = [EvaluationResult(self.n, c[b, : self.n].copy(), c[b, self.n:].copy()) for b in range(len(pts))]
        t1 = time.perf_counter()
        evals = len(pts) * repeat
        mc = self._mults
        delta = MultCounter(mc.stage1_powers - before.stage1_powers, mc.stage1_factors - before.stage1_factors,
                            mc.stage2 - before.stage2, mc.speelpenning - before.speelpenning, mc.stage3 - before.stage3)
        rep = BatchReport(evals, t1 - t0, (t1 - t0) / evals if evals else 0.0, delta)
        return BatchResult(results, rep)

    # ---- device path (torch tensors)
    def _dev_tensor(self, what: str, t, shape, dtype: str = "float64"):
        """The kernels take raw pointers: reject anything but a contiguous CUDA tensor of the exact
        shape and dtype on this context's device (a float32 or strided view would be read past its
        end)."""
        import torch
        want = {"float64": torch.float64, "int32": torch.int32}[dtype]
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{what}: expected a torch.Tensor on cuda:{self.device}")
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{what}: shape {tuple(t.shape)} != {tuple(shape)}")
        if t.dtype != want:
            raise TypeError(f"{what}: dtype {t.dtype} != {want}")
        if t.device.type != "cuda" or t.device.index != self.device:
            raise ValueError(f"{what}: tensor on {t.device}, context on cuda:{self.device}")
        if not t.is_contiguous():
            raise ValueError(f"{what}: tensor must be contiguous")
        return t.data_ptr()

    def evaluate_device(self, points, out, precision: str = "dd", order: str | None = None, stream=None,
                        validate: bool = False) -> None:
        """Asynchronous evaluation of device-resident points. points/out: contiguous float64 CUDA
        tensors on this context's device, [B, n, W] / [B, n + n*n, W]; stream: a torch.cuda.Stream,
        a raw cudaStream_t int, or None (torch's current stream). validate=True checks the points
        first and raises ValueError before anything is written when a coordinate is non-finite
        (PJ_VALIDATE: one stream synchronisation), like ref src/engine.cpp:183-188."""
        W = 2 if precision == "d" else 4
        B = int(points.shape[0])
        pp = self._dev_tensor("evaluate_device: points", points, (B, self.n, W))
        po = self._dev_tensor("evaluate_device: out", out, (B, self.n + self.n * self.n, W))
        flags = _flags(precision, order) | (_lib.PJ_VALIDATE if validate else 0)
        check(lib().pj_evaluate(self._h, flags, pp, B, po, ctypes.c_void_p(self._stream(stream, points))))

    def nonfinite_seen(self, stream=None) -> bool:
        if hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        seen = ctypes.c_int(0)
        check(lib().pj_nonfinite_seen(self._h, ctypes.c_void_p(stream or 0), ctypes.byref(seen)))
        return bool(seen.value)

    # ---- Newton corrector (csrc/newton.cu)
    def newton_host(self, points: np.ndarray, precision: str = "dd", iters: int = 1, target: np.ndarray | None = None,
                    order: str | None = None, out: np.ndarray | None = None, norms: np.ndarray | None = None,
                    status: np.ndarray | None = None):
        """`iters` Newton steps x <- x + J(x)^-1 (y - f(x)) per point, on the GPU.
        points (and target y, optional; absent = the roots of f): [B, n, W] float64.
        Returns (points_out [B, n, W], norms [B, 2] = max-norms of y - f and of the last step,
        status [B] int32: 0 ok, 1 singular Jacobian, 2 non-finite result, 3 mixed solve not converged).
        precision: 'd', 'dd' or 'mixed' (dd points; the Jacobian factored in complex double and refined
        with dd residuals — faster, for Jacobians that are not ill-conditioned). out / norms / status may be
        preallocated (page-locked buffers give full H2D / compute / D2H overlap)."""
        W = 2 if precision == "d" else 4
        pts = np.ascontiguousarray(points, np.float64)
        if pts.ndim != 3 or pts.shape[1:] != (self.n, W):
            raise ValueError("newton: point dimension mismatch")
        tg = None
        if target is not None:
            tg = np.ascontiguousarray(target, np.float64)
            if tg.shape != pts.shape:
                raise ValueError("newton: target shape mismatch")
        B = pts.shape[0]
        if out is None:
            out = np.empty_like(pts)
        if norms is None:
            norms = np.empty((B, 2), np.float64)
        if status is None:
            status = np.empty(B, np.int32)
        for a, shp, dt in ((out, pts.shape, np.float64), (norms, (B, 2), np.float64), (status, (B,), np.int32)):
            if a.shape != shp or a.dtype != dt or not a.flags.c_contiguous:
                raise ValueError("newton: output buffer must be C-contiguous %s of shape %s" % (np.dtype(dt), shp))
        check(lib().pj_newton_host(self._h, _nflags(precision, order), pts.ctypes.data,
                                   tg.ctypes.data if tg is not None else None, B, iters, out.ctypes.data,
                                   norms.ctypes.data, status.ctypes.data))
        self._add_tally(B * iters)
        return out, norms, status

    @staticmethod
    def _stream(stream, like):
        if stream is None:
            import torch
            return torch.cuda.current_stream(like.device).cuda_stream
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else stream

    def newton_solve_device(self, evals, points, out, precision: str = "dd", target=None, norms=None, status=None,
                            stream=None) -> None:
        """Asynchronous Newton solve from device-resident evaluator output (pj_newton_solve)."""
        W = 2 if precision == "d" else 4
        B = int(points.shape[0])
        n = self.n
        what = "newton_solve_device"
        pe = self._dev_tensor(what + ": evals", evals, (B, n + n * n, W))
        pp = self._dev_tensor(what + ": points", points, (B, n, W))
        po = self._dev_tensor(what + ": out", out, (B, n, W))
        pt = self._dev_tensor(what + ": target", target, (B, n, W)) if target is not None else None
        pn = self._dev_tensor(what + ": norms", norms, (B, 2)) if norms is not None else None
        ps = self._dev_tensor(what + ": status", status, (B,), "int32") if status is not None else None
        check(lib().pj_newton_solve(self._h, _nflags(precision, None), pe, pp, pt, B, po, pn, ps,
                                    ctypes.c_void_p(self._stream(stream, points))))

    def newton_step_device(self, points, work, out, precision: str = "dd", target=None, norms=None, status=None,
                           order: str | None = None, stream=None) -> None:
        """Asynchronous evaluate + Newton solve (pj_newton_step); work: [B, n + n*n, W]."""
        W = 2 if precision == "d" else 4
        B = int(points.shape[0])
        n = self.n
        what = "newton_step_device"
        pp = self._dev_tensor(what + ": points", points, (B, n, W))
        pw = self._dev_tensor(what + ": work", work, (B, n + n * n, W))
        po = self._dev_tensor(what + ": out", out, (B, n, W))
        pt = self._dev_tensor(what + ": target", target, (B, n, W)) if target is not None else None
        pn = self._dev_tensor(what + ": norms", norms, (B, 2)) if norms is not None else None
        ps = self._dev_tensor(what + ": status", status, (B,), "int32") if status is not None else None
        check(lib().pj_newton_step(self._h, _nflags(precision, order), pp, pt, B, pw, po, pn, ps,
                                   ctypes.c_void_p(self._stream(stream, points))))

    # ---- index maps (bit-exact with the reference)
    def slot_targets(self, s: int) -> np.ndarray:
        out = np.empty(self.k + 1, np.int64)
        check(lib().pj_slot_targets(self._h, s, out.ctypes.data))
        return out

    def zero_mask(self) -> np.ndarray:
        ln = lib().pj_zero_mask(self._h, None, 0)
        if ln < 0:
            check(_lib.PJ_EINVAL)
        out = np.empty(ln, np.int64)
        lib().pj_zero_mask(self._h, out.ctypes.data, ln)
        return out

    # ---- launch shape
    def set_launch(self, precision: str, threads: int = 0, tile_points: int = 0, order: str | None = None,
                   newton: bool = False) -> None:
        """Override the launch shape of the evaluation kernel (or, newton=True, the Newton solve)."""
        f = (_nflags(precision, order) | _lib.PJ_OP_NEWTON) if newton else _flags(precision, order)
        check(lib().pj_set_launch(self._h, f, threads, tile_points))

    def set_variant(self, variant: int, precision: str = "dd", newton: bool = False) -> None:
        """Kernel choice (pj_set_kernel_variant) for complex double ("d") or the fast dd order:
        0 auto, -1 generic, 1 k-specialised, 3 warp-specialised (dd, d <= 2, m <= 32, n <= 64,
        k <= 12); newton=True: the Newton solve (-1 column kernel,
        1 panel kernel for n <= 32)."""
        f = _flags(precision, None) | (_lib.PJ_OP_NEWTON if newton else 0)
        check(lib().pj_set_kernel_variant(self._h, f, variant))

    def launch(self, precision: str, order: str | None = None, newton: bool = False):
        t, tp, b, var = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        sm = ctypes.c_int64()
        f = (_nflags(precision, order) | _lib.PJ_OP_NEWTON) if newton else _flags(precision, order)
        check(lib().pj_get_launch(self._h, f, ctypes.byref(t), ctypes.byref(tp),
                                  ctypes.byref(b), ctypes.byref(sm), ctypes.byref(var)))
        return dict(threads=t.value, tile_points=tp.value, blocks=b.value, smem_bytes=sm.value, variant=var.value)


def fp64_pipe_rates(device: int = 0) -> dict:
    """Issue rate of the FP64 pipe (lane operations / s) for DFMA, DADD and DMUL (pj_fp64_pipe_probe)."""
    v = (ctypes.c_double * 3)()
    check(lib().pj_fp64_pipe_probe(device, ctypes.addressof(v)))
    return {"dfma": v[0], "dadd": v[1], "dmul": v[2]}


def fp64_peak_tflops(device: int = 0) -> float:
    v = ctypes.c_double(0)
    check(lib().pj_fp64_peak_probe(device, ctypes.byref(v)))
    return v.value

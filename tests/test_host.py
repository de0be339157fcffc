"""Host-side logic of the product library (CPU, no GPU): the C ABI loads and exports every
symbol include/polyjac_b200.h declares; generator, validation, packing v2 and the index maps
are bit-exact with the reference; error behaviour mirrors the reference's exceptions."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1201_0499_b200 as pj
from conftest import ROOT, sysd_of
from oracle import oracle as O
from paper_1201_0499_b200 import _lib
from paper_1201_0499_b200.sharding import shard_range

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "polyjac_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(pj_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    syms = header_symbols()
    assert len(syms) >= 18
    L = ctypes.CDLL(_lib.SO_PATH)
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(_lib.EXPORTS) == syms


def test_library_is_sm100a():
    import subprocess
    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.SO_PATH], capture_output=True, text=True)
    assert "sm_100a" in r.stdout


def test_version_string():
    assert b"sm_100a" in _lib.lib().pj_version()


@needs_ref
@pytest.mark.parametrize("shape,seed", [((32, 32, 8, 2), 7), ((64, 64, 16, 10), 7), ((24, 7, 5, 11), 77),
                                        ((4, 1, 1, 1), 1), ((40, 40, 20, 3), 9), ((300, 1, 1, 1), 3)])
def test_random_system_bit_identical_to_reference(shape, seed):
    s = pj.random_system(*shape, seed)
    r = O.ref_random_system(*shape, seed)
    assert np.array_equal(s.positions.reshape(-1), r["pos"])
    assert np.array_equal(s.exponents.reshape(-1), r["exps"])
    assert np.array_equal(s.coeffs.view(np.uint64), r["coeffs"].view(np.uint64))


@needs_ref
def test_random_points_and_ranges_bit_identical():
    full = O.ref_random_points(32, 50, 11)
    mine = pj.random_points(32, 50, 11).view(np.float64).reshape(50, 32, 2)
    assert np.array_equal(full.view(np.uint64), mine.view(np.uint64))
    from paper_1201_0499_b200.sharding import shard_points
    parts = [shard_points(32, 50, 11, 3, r).view(np.float64).reshape(-1, 32, 2) for r in range(3)]
    assert np.array_equal(np.concatenate(parts).view(np.uint64), full.view(np.uint64))
    # the CLI's single point convention (ref tools/main.cpp:17,77)
    p = pj.random_point(32, 7 ^ 0x9e3779b97f4a7c15)
    assert np.array_equal(p.view(np.float64), O.ref_random_points(32, 1, 7 ^ 0x9e3779b97f4a7c15).reshape(-1))


def test_random_system_argument_errors():
    for args in [(0, 1, 1, 1), (2, 0, 1, 1), (2, 1, 3, 1), (2, 1, 0, 1), (2, 1, 1, 0), (2, 1, 1, 256)]:
        with pytest.raises(ValueError):
            pj.random_system(*args, 1)


def _mutations():
    base = pj.random_system(6, 3, 3, 4, 9)
    out = []

    def mut(f):
        s = pj.PolynomialSystem(base.n, base.m, base.k, base.d, base.positions.copy(), base.exponents.copy(),
                                base.coeffs.copy())
        f(s)
        out.append(s)

    mut(lambda s: s.coeffs.__setitem__((4, slice(None)), 0.0))                     # zero coefficient
    mut(lambda s: s.coeffs.__setitem__((2, 0), np.inf))                            # non-finite
    mut(lambda s: s.positions.__setitem__((5, 1), s.positions[5, 0]))             # not increasing
    mut(lambda s: s.positions.__setitem__((1, 2), 6))                             # out of range
    mut(lambda s: s.exponents.__setitem__((7, 0), 5))                             # exponent > d
    mut(lambda s: s.exponents.__setitem__((7, 0), 0))                             # exponent < 1
    return base, out


@needs_ref
def test_validation_matches_reference():
    base, bad = _mutations()
    assert pj.validate_system(base).ok()
    for s in bad:
        rep = pj.validate_system(s)
        nref, msg = O.ref_validate(sysd_of(s))
        assert len(rep.violations) == nref > 0
        assert rep.violations[0].describe() == msg
        with pytest.raises(ValueError):
            pj.EvaluationContext(s, device=-1)


def test_layout_rejects_n_over_256():
    s = pj.random_system(300, 1, 1, 1, 3)
    assert pj.validate_system(s).ok()
    with pytest.raises(ValueError, match="n > 256"):
        pj.EvaluationContext(s, device=-1)


def test_term_count_mismatch_rejected():
    t = pj.Term(1 + 0j, pj.MonomialSupport([0], [1]))
    s = pj.PolynomialSystem.from_terms(2, 1, 1, 1, [t])
    assert not pj.validate_system(s).ok()


def test_grid_config_validated():
    s = pj.random_system(4, 2, 2, 2, 3)
    with pytest.raises(ValueError):
        pj.EvaluationContext(s, pj.GridConfig(0, 1), device=-1)
    with pytest.raises(ValueError):
        pj.EvaluationContext(s, pj.GridConfig(32, -1), device=-1)
    assert pj.EvaluationContext(s, pj.GridConfig(32, 0), device=-1).grid().workers >= 1


def test_mons_slot_known_answers_and_errors():
    # ref tests/test_packing.cpp:78-86
    assert pj.mons_value_slot(0, 32, 32) == 0
    assert pj.mons_deriv_slot(0, 0, 32, 32) == 32
    assert pj.mons_value_slot(33, 32, 32) == 1057
    with pytest.raises(IndexError):
        pj.mons_value_slot(1024, 32, 32)
    with pytest.raises(IndexError):
        pj.mons_deriv_slot(0, 32, 32, 32)
    with pytest.raises(IndexError):
        pj.mons_deriv_slot(0, -1, 32, 32)


@needs_ref
def test_mons_slot_exhaustive_vs_reference():
    for n, m in [(3, 1), (5, 4), (32, 32)]:
        for s in range(-1, n * m + 1):
            for var in (-1, 0, n - 1, n):
                want = O.ref_mons_slot(s, "deriv", var, n, m)
                try:
                    got = pj.mons_deriv_slot(s, var, n, m)
                except IndexError:
                    got = -1
                assert got == want


SHAPES = [(4, 1, 1, 1), (4, 4, 2, 3), (8, 3, 8, 2), (16, 16, 9, 2), (32, 32, 9, 2), (32, 22, 9, 2),
          (32, 48, 16, 10), (40, 40, 20, 3), (10, 40, 4, 3), (12, 5, 6, 4), (64, 64, 16, 10)]


@needs_ref
@pytest.mark.parametrize("shape", SHAPES)
def test_gather_map_regenerates_reference_index_maps(shape):
    """The device gather map's complement is the reference zero mask and the per-monomial
    targets are stage2_slot_targets — bit-exact (ref src/packing.cpp:54-72, kernels.cpp:129-137)."""
    s = pj.random_system(*shape, 31000 + shape[0] * 7 + shape[2])
    S = sysd_of(s)
    ctx = pj.EvaluationContext(s, device=-1)
    assert np.array_equal(ctx.zero_mask(), O.ref_zero_mask(S))
    n, m, k = shape[:3]
    t = np.stack([ctx.slot_targets(i) for i in range(n * m)])
    assert np.array_equal(t, O.ref_slot_targets(S))
    assert len(ctx.zero_mask()) == (n * n + n) * m - n * m * (k + 1)


@needs_ref
def test_layout_info_footprint():
    s = pj.random_system(32, 32, 9, 2, 7)
    info = pj.EvaluationContext(s, device=-1).layout_info()
    assert info["footprint_bytes"] == 18432  # ref tests/test_packing.cpp:57-64


def test_mult_counts_closed_form():
    n, m, k, d = 8, 5, 4, 6
    ctx = pj.EvaluationContext(pj.random_system(n, m, k, d, 17), device=-1)
    t = ctx._tally(25)
    assert t.total() == (n * (d - 2) + n * m * (k - 1) + n * m * (5 * k - 4)) * 25
    assert t.stage3 == 0 and t.stage1_powers == n * (d - 2) * 25 and t.speelpenning == n * m * (3 * k - 6) * 25


def test_host_only_context_refuses_evaluation():
    ctx = pj.EvaluationContext(pj.random_system(4, 2, 2, 2, 8), device=-1)
    with pytest.raises(ValueError, match="host-only"):
        ctx.evaluate_host(np.zeros((1, 4, 2)), "d")


def test_shard_range_partitions():
    for total in (0, 1, 7, 65536, 1 << 20):
        for ws in (1, 2, 3, 8):
            rs = [shard_range(total, ws, r) for r in range(ws)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_newton_and_launch_argument_errors_host_only():
    L = _lib.lib()
    ctx = pj.EvaluationContext(pj.random_system(4, 2, 2, 2, 8), device=-1)
    with pytest.raises(ValueError, match="host-only"):
        ctx.newton_host(np.zeros((1, 4, 4)), "dd")
    with pytest.raises(ValueError, match="iterations"):
        ctx.newton_host(np.zeros((1, 4, 4)), "dd", iters=0)
    with pytest.raises(ValueError, match="dimension"):
        ctx.newton_host(np.zeros((1, 3, 4)), "dd")
    with pytest.raises(ValueError, match="precision"):
        ctx.newton_host(np.zeros((1, 4, 4)), "qd")
    # C ABI: null buffers, negative batch, unknown precision flag; batch 0 is a no-op
    h = ctx._h
    assert L.pj_newton_solve(h, _lib.PJ_PREC_DD, None, None, None, 1, None, None, None, None) == _lib.PJ_EINVAL
    assert L.pj_newton_solve(h, _lib.PJ_PREC_DD, None, None, None, -1, None, None, None, None) == _lib.PJ_EINVAL
    assert L.pj_newton_solve(h, 7, None, None, None, 1, None, None, None, None) == _lib.PJ_EINVAL
    assert L.pj_newton_solve(h, _lib.PJ_PREC_DD, None, None, None, 0, None, None, None, None) == _lib.PJ_OK
    assert L.pj_newton_step(h, _lib.PJ_PREC_D, None, None, 2, None, None, None, None, None) == _lib.PJ_EINVAL
    # launch overrides: thread counts must be multiples of 32 up to 384
    for bad in (-32, 33, 416):
        assert L.pj_set_launch(h, _lib.PJ_PREC_DD, bad, 0) == _lib.PJ_EINVAL
    assert L.pj_set_kernel_variant(h, _lib.PJ_PREC_DD | _lib.PJ_ORDER_REF, 1) == _lib.PJ_EINVAL


def test_context_options_validated():
    s = pj.random_system(4, 2, 2, 2, 8)
    desc, keep = s._desc()
    h = ctypes.c_void_p()
    assert _lib.lib().pj_ctx_create_ex(ctypes.byref(desc), -1, 0x80, ctypes.byref(h)) == _lib.PJ_EINVAL
    assert "option" in _lib.last_error()
    assert _lib.lib().pj_ctx_create_ex(ctypes.byref(desc), -1, _lib.PJ_CTX_WIDE, ctypes.byref(h)) == _lib.PJ_OK
    _lib.lib().pj_ctx_destroy(h)


@needs_ref
@pytest.mark.parametrize("shape", [(32, 32, 8, 2), (64, 64, 16, 10), (8, 3, 3, 5), (4, 4, 1, 1), (40, 40, 20, 3)])
def test_layout_export_bit_identical_to_build_layout(shape):
    # EvaluationContext::layout() (ref include/polyjac/engine.hpp:100) through pj_layout_export
    s = pj.random_system(*shape, 77)
    lay = pj.EvaluationContext(s, device=-1).layout()
    n, m, k, d = shape
    nm = n * m
    rp, re = np.empty(nm * k, np.uint8), np.empty(nm * k, np.uint8)
    rc = np.empty(((k + 1) * nm, 2), np.float64)
    sd = sysd_of(s)
    assert O.ref().ref_build_layout(n, m, k, d, sd["pos"], sd["exps"], sd["coeffs"], rp, re, rc) == 0
    assert np.array_equal(lay.positions, rp) and np.array_equal(lay.exponents, re)
    assert np.array_equal(lay.coeffs.view(np.float64).reshape(-1, 2).view(np.uint64), rc.view(np.uint64))
    assert lay.footprint_bytes() == 2 * nm * k
    assert lay.position(5, 0) == rp[5 * k] and lay.value_coeff(3) == complex(*rc[k * nm + 3])


def test_structural_zeros_match_the_zero_mask():
    # Jacobian entry (p, v) is a structural zero iff none of its m derivative slots is claimed
    s = pj.random_system(10, 4, 3, 3, 33)
    ctx = pj.EvaluationContext(s, device=-1)
    mask = np.zeros(100, np.uint8)
    cnt = pj._lib.lib().pj_structural_zeros(ctx._h, mask.ctypes.data)
    claimed = np.zeros((10, 10), bool)
    for sidx in range(40):
        for v in s.positions[sidx]:
            claimed[sidx // 4, v] = True
    assert cnt == int((~claimed).sum()) and np.array_equal(mask.reshape(10, 10).astype(bool), ~claimed)

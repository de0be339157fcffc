"""Ragged systems: non-uniform m per polynomial and k per term (second half).

The reference's data model is uniform (ref include/polyjac/system.hpp:14-42), so the ragged
contract is pinned three ways:
  * the oracle's ragged restatement (oracle.cpp: evaluate_one_ragged) reproduces the uniform
    oracle bit for bit on uniform systems written in ragged form — and the uniform oracle is
    pinned to the unmodified reference's bits (tests/test_oracle.py);
  * the oracle is within 1e-30 * sum|terms| (dd) of the mpmath truth on tests/golden/ragged
    (gen_ragged_golden.py: shapes crossing the 32-monomial chunk, k = 1 / 2 special cases, d = 1);
  * on the GPU (generic kernel, RAG = true): complex double and dd reference order bit-exact with
    the oracle; dd fast order within the tolerance of mpmath and of the oracle; structural zeros
    exact +0; a uniform system in ragged form gives the uniform context's bits (d, dd ref).
Validation follows validate_system's wording per term (ref src/system.cpp:21-64).
"""
import glob
import os

import numpy as np
import pytest

import paper_1201_0499_b200 as pj
from conftest import DD_TOL, GOLDEN, dd_err, dd_rel, sysd_of
from oracle import oracle as O

RAGGED_GOLDEN = sorted(glob.glob(os.path.join(GOLDEN, "ragged", "*.npz")))


def load_ragged(path):
    z = np.load(path)
    S = dict(n=int(z["n"]), d=int(z["d"]), row_off=z["row_off"].astype(np.int32),
             term_off=z["term_off"].astype(np.int32), pos=z["pos"].astype(np.int32),
             exps=z["exps"].astype(np.int32), coeffs=z["coeffs"])
    return S, z


def system_of(S):
    return pj.RaggedSystem(S["n"], S["d"], S["row_off"], S["term_off"], S["pos"], S["exps"], S["coeffs"])


def d_points(pdd):
    return np.ascontiguousarray(pdd[..., [0, 2]])


# ------------------------------------------------------------------ oracle pins (CPU)
@pytest.mark.parametrize("path", RAGGED_GOLDEN, ids=lambda p: p.split("/")[-1])
def test_oracle_ragged_dd_matches_mpmath(path):
    S, z = load_ragged(path)
    got = O.evaluate_ragged("dd", S, z["points_dd"])
    assert dd_rel(got, z["truth_dd"], z["magsum"]) <= DD_TOL


@pytest.mark.parametrize("path", RAGGED_GOLDEN, ids=lambda p: p.split("/")[-1])
def test_oracle_ragged_d_near_mpmath(path):
    S, z = load_ragged(path)
    got = O.evaluate_ragged("d", S, d_points(z["points_dd"]))
    t = z["truth_dd"]
    err = np.maximum(np.abs(got[..., 0] - (t[..., 0] + t[..., 1])), np.abs(got[..., 1] - (t[..., 2] + t[..., 3])))
    ms = z["magsum"]
    assert np.all(got[ms == 0] == 0)
    assert float(np.max(err[ms > 0] / ms[ms > 0])) <= 1e-14


@pytest.mark.parametrize("shape", [(6, 4, 1, 3), (6, 4, 2, 3), (8, 5, 3, 4), (10, 40, 4, 3), (32, 32, 8, 2)])
def test_oracle_ragged_equals_uniform_oracle(shape):
    n, m, k, d = shape
    s = pj.random_system(n, m, k, d, 17 + n + k)
    r = pj.RaggedSystem.from_uniform(s)
    z = pj.random_points(n, 3, 5)
    p2 = np.stack([z.real, z.imag], -1)
    pdd = pj.to_dd(z)
    pdd[..., 1] = pdd[..., 0] * 2.0 ** -55
    for prec, pts in (("d", p2), ("dd", pdd)):
        a = O.evaluate_ragged(prec, r.as_dict(), pts)
        b = O.evaluate(prec, sysd_of(s), pts)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), prec


def test_oracle_ragged_d_pinned_to_reference_through_uniform():
    # the chain of pins: ragged oracle == uniform oracle == the unmodified reference (double)
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    s = pj.random_system(12, 7, 3, 3, 91)
    z = pj.random_points(12, 4, 92)
    p2 = np.stack([z.real, z.imag], -1)
    a = O.evaluate_ragged("d", pj.RaggedSystem.from_uniform(s).as_dict(), p2)
    assert np.array_equal(a.view(np.uint64), O.ref_evaluate(sysd_of(s), p2).view(np.uint64))


# ------------------------------------------------------------------ host side (CPU)
def test_generator_is_deterministic_and_valid():
    a = pj.random_ragged_system(16, (3, 40), (1, 9), 4, 123)
    b = pj.random_ragged_system(16, (3, 40), (1, 9), 4, 123)
    for f in ("row_off", "term_off", "positions", "exponents", "coeffs"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    assert pj.validate_ragged_system(a).ok()
    m = np.diff(a.row_off)
    k = np.diff(a.term_off)
    assert m.min() >= 3 and m.max() <= 40 and k.min() >= 1 and k.max() <= 9
    assert a.exponents.min() >= 1 and a.exponents.max() <= 4
    # equal bounds reproduce the uniform generator's per-term draws only in shape, not stream
    u = pj.random_ragged_system(8, (5, 5), (3, 3), 2, 1)
    assert np.all(np.diff(u.row_off) == 5) and np.all(np.diff(u.term_off) == 3)


@pytest.mark.parametrize("bad,msg", [
    (lambda r: r.coeffs.__setitem__(3, 0.0), "polynomial 0, monomial 3: zero coefficient"),
    (lambda r: r.coeffs.__setitem__((2, 0), np.nan), "polynomial 0, monomial 2: non-finite coefficient"),
    (lambda r: r.exponents.__setitem__(0, 9), "polynomial 0, monomial 0: exponent out of range [1,d]"),
    (lambda r: r.positions.__setitem__(0, 99), "polynomial 0, monomial 0: variable index out of range [0,n-1]"),
])
def test_ragged_validation_wording(bad, msg):
    r = pj.random_ragged_system(6, (4, 4), (2, 2), 3, 7)
    if "zero coefficient" in msg:
        r.coeffs[3] = 0.0
    else:
        bad(r)
    rep = pj.validate_ragged_system(r)
    assert not rep.ok() and rep.violations[0].describe() == msg
    with pytest.raises(ValueError, match="invalid system"):
        pj.EvaluationContext(r, device=-1)


def test_ragged_shape_rules():
    r = pj.RaggedSystem.from_polynomials(3, 2, [
        [pj.Term(1 + 0j, pj.MonomialSupport([0, 2], [1, 2]))],
        [pj.Term(2 + 1j, pj.MonomialSupport([1], [1])), pj.Term(0.5j, pj.MonomialSupport([0, 1, 2], [1, 1, 1]))],
        [pj.Term(-1 + 0j, pj.MonomialSupport([2, 1], [1, 1]))],
    ])
    assert pj.validate_ragged_system(r).violations[0].describe() == \
        "polynomial 2, monomial 0: positions not strictly increasing"
    empty = pj.RaggedSystem.from_polynomials(2, 2, [[pj.Term(1 + 0j, pj.MonomialSupport([0], [1]))], []])
    assert pj.validate_ragged_system(empty).violations[0].describe() == "polynomial 1: m must be at least 1"
    big = pj.RaggedSystem.from_polynomials(2, 2, [[pj.Term(1 + 0j, pj.MonomialSupport([0, 1, 1], [1, 1, 1]))],
                                                  [pj.Term(1 + 0j, pj.MonomialSupport([0], [1]))]])
    assert "k exceeds n" in [v.rule for v in [pj.validate_ragged_system(big).violations[0]]][0]
    nok = pj.RaggedSystem.from_polynomials(2, 2, [[pj.Term(1 + 0j, pj.MonomialSupport([], []))],
                                                  [pj.Term(1 + 0j, pj.MonomialSupport([0], [1]))]])
    assert pj.validate_ragged_system(nok).violations[0].describe() == \
        "polynomial 0, monomial 0: k must be at least 1"


def test_ragged_host_context_maps():
    r = pj.random_ragged_system(20, (1, 50), (1, 7), 3, 44)
    ctx = pj.EvaluationContext(r, device=-1)
    info = ctx.layout_info()
    assert info["m"] == int(np.diff(r.row_off).max()) and info["k"] == int(np.diff(r.term_off).max())
    assert info["footprint_bytes"] == 2 * int(r.term_off[-1])
    # structural zeros: (p, v) with v in no term of row p
    want = np.ones((20, 20), bool)
    for p in range(20):
        for t in range(r.row_off[p], r.row_off[p + 1]):
            want[p, r.positions[r.term_off[t]:r.term_off[t + 1]]] = False
    got = ctx._structural_zeros() - 20
    assert np.array_equal(got, np.nonzero(want.reshape(-1))[0])
    # multiplication tally: the closed form per term
    k = np.diff(r.term_off).astype(np.int64)
    sp = np.where(k >= 3, 3 * k - 6, 0)
    mc = ctx._tally(3)
    assert mc.stage1_powers == 3 * 20 * 1 and mc.stage1_factors == 3 * int(np.sum(k - 1))
    assert mc.speelpenning == 3 * int(sp.sum()) and mc.stage2 == 3 * int(np.sum(sp + 2 * k + 2))
    # the uniform-layout exports are not defined for a ragged system
    with pytest.raises(ValueError):
        ctx.layout()
    with pytest.raises(ValueError):
        ctx.zero_mask()
    with pytest.raises(ValueError):
        ctx.slot_targets(0)


def test_ragged_byte_cap_and_wide():
    r = pj.random_ragged_system(300, (1, 2), (1, 3), 2, 8)
    with pytest.raises(ValueError, match="n > 256"):
        pj.EvaluationContext(r, device=-1)
    pj.EvaluationContext(r, device=-1, wide=True)


# ------------------------------------------------------------------ device parity
def check_device(ctx, S, pdd, truth=None, magsum=None):
    want_dd, ms = O.evaluate_ragged("dd", S, pdd, magsum=True)
    got_ref = ctx.evaluate_dd(pdd, order="ref")
    assert np.array_equal(got_ref.view(np.uint64), want_dd.view(np.uint64)), "dd reference order != oracle"
    got = ctx.evaluate_dd(pdd)
    assert dd_rel(got, want_dd, ms) <= DD_TOL
    if truth is not None:
        assert dd_rel(got, truth, magsum) <= DD_TOL
        assert dd_rel(got_ref, truth, magsum) <= DD_TOL
    p2 = d_points(pdd)
    got_d = ctx.evaluate_host(p2, "d")
    want_d = O.evaluate_ragged("d", S, p2)
    assert np.array_equal(got_d.view(np.uint64), want_d.view(np.uint64)), "complex double != oracle"
    assert ctx.masked_slots_clean()


@pytest.mark.gpu
@pytest.mark.parametrize("path", RAGGED_GOLDEN, ids=lambda p: p.split("/")[-1])
def test_ragged_golden_on_device(path, gpu):
    S, z = load_ragged(path)
    ctx = pj.EvaluationContext(system_of(S))
    check_device(ctx, S, z["points_dd"], z["truth_dd"], z["magsum"])


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(32, (16, 48), (2, 12), 2), (24, (1, 70), (1, 16), 5), (40, (30, 34), (6, 10), 3)])
def test_ragged_random_batch_on_device(shape, gpu):
    n, mr, kr, d = shape
    r = pj.random_ragged_system(n, mr, kr, d, 1000 + n)
    z = pj.random_points(n, 300, 77) * 0.9
    pdd = pj.to_dd(z)
    pdd[..., 1] = pdd[..., 0] * 2.0 ** -56
    pdd[..., 3] = -pdd[..., 2] * 2.0 ** -57
    check_device(pj.EvaluationContext(r), r.as_dict(), pdd)


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(32, 32, 8, 2), (10, 40, 4, 3), (6, 4, 1, 3), (6, 4, 2, 3)])
def test_uniform_as_ragged_matches_uniform_context(shape, gpu):
    n, m, k, d = shape
    s = pj.random_system(n, m, k, d, 7)
    cu = pj.EvaluationContext(s)
    cr = pj.EvaluationContext(pj.RaggedSystem.from_uniform(s))
    z = pj.random_points(n, 64, 11)
    p2 = np.stack([z.real, z.imag], -1)
    assert np.array_equal(cr.evaluate_host(p2, "d").view(np.uint64), cu.evaluate_host(p2, "d").view(np.uint64))
    pdd = pj.to_dd(z)
    pdd[..., 1] = pdd[..., 0] * 2.0 ** -57
    a, b = cr.evaluate_dd(pdd, order="ref"), cu.evaluate_dd(pdd, order="ref")
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    want, ms = O.evaluate("dd", sysd_of(s), pdd, magsum=True)
    assert dd_rel(cr.evaluate_dd(pdd), want, ms) <= DD_TOL


@pytest.mark.gpu
def test_ragged_wide_on_device(gpu):
    r = pj.random_ragged_system(300, (1, 3), (1, 4), 3, 301)
    z = pj.random_points(300, 6, 302) * 0.95
    pdd = pj.to_dd(z)
    check_device(pj.EvaluationContext(r, wide=True), r.as_dict(), pdd)


@pytest.mark.gpu
def test_ragged_newton_step_bit_exact(gpu):
    # f1 on a ragged system: the solve only sees the evaluator's output, so one step in the dd
    # reference order equals the oracle's evaluation followed by the oracle's solve
    r = pj.random_ragged_system(16, (8, 24), (1, 6), 2, 5)
    ctx = pj.EvaluationContext(r)
    z = pj.random_points(16, 40, 6) * 0.8
    pdd = pj.to_dd(z)
    xn, norms, status = ctx.newton_host(pdd, "dd", iters=1, order="ref")
    ev = O.evaluate_ragged("dd", r.as_dict(), pdd)
    want_x, want_norms, want_st = O.newton_solve("dd", 16, ev, pdd)
    assert np.array_equal(status, want_st)
    assert np.array_equal(xn.view(np.uint64), want_x.view(np.uint64))
    p2 = d_points(pdd)
    xd, _, sd = ctx.newton_host(p2, "d", iters=1)
    wd, _, wsd = O.newton_solve("d", 16, O.evaluate_ragged("d", r.as_dict(), p2), p2)
    assert np.array_equal(sd, wsd) and np.array_equal(xd.view(np.uint64), wd.view(np.uint64))


@pytest.mark.gpu
def test_ragged_device_tensor_path(gpu):
    import torch
    r = pj.random_ragged_system(12, (2, 40), (1, 5), 4, 9)
    ctx = pj.EvaluationContext(r)
    z = pj.random_points(12, 100, 10)
    pdd = pj.to_dd(z)
    x = torch.from_numpy(pdd).cuda()
    out = torch.empty((100, 12 + 144, 4), dtype=torch.float64, device="cuda")
    ctx.evaluate_device(x, out, "dd", order="ref")
    torch.cuda.synchronize()
    want = O.evaluate_ragged("dd", r.as_dict(), pdd)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want.view(np.uint64))
    assert float(np.max(dd_err(out.cpu().numpy(), want))) == 0.0

"""The oracle is pinned before it is trusted (CPU, no GPU).

* complex double: the oracle's restatement reproduces the UNMODIFIED reference bit for bit
  (oracle/_ref, compiled from /root/reference/proj/src) and the committed reference outputs
  in tests/golden (ref_d);
* complex double-double: within 1e-30 * sum|terms| of the mpmath truth in tests/golden,
  exact +0 on structural zeros;
* the reference's own known-answer tests (ref tests/test_kernels.cpp, test_packing.cpp,
  test_engine.cpp) restated: integer-valued answers are exact in any precision.
"""
import numpy as np
import pytest

from conftest import DD_TOL, dd_rel, golden_cases, load_golden
from oracle import oracle as O


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: p.split("/")[-1])
def test_oracle_double_matches_reference_golden_bits(path):
    S, z = load_golden(path)
    got = O.evaluate("d", S, z["points_d"])
    assert np.array_equal(got.view(np.uint64), z["ref_d"].view(np.uint64))


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: p.split("/")[-1])
def test_oracle_dd_matches_mpmath_truth(path):
    S, z = load_golden(path)
    got = O.evaluate("dd", S, z["points_dd"])
    assert dd_rel(got, z["truth_dd"], z["magsum"]) <= DD_TOL


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: p.split("/")[-1])
def test_oracle_magsum_matches_truth_scale(path):
    S, z = load_golden(path)
    _, ms = O.evaluate("dd", S, z["points_dd"], magsum=True)
    nz = z["magsum"] > 0
    assert np.array_equal(ms > 0, nz)
    assert np.allclose(ms[nz], z["magsum"][nz], rtol=1e-12)


needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")


@needs_ref
@pytest.mark.parametrize("shape", [(32, 32, 9, 2), (32, 32, 16, 10), (8, 3, 3, 5), (4, 4, 1, 1), (6, 4, 2, 3),
                                   (40, 40, 20, 3), (4, 1, 1, 255), (12, 5, 6, 4)])
def test_oracle_double_bit_exact_vs_reference_library(shape):
    n, m, k, d = shape
    S = O.ref_random_system(n, m, k, d, 7000 + n + k + d)
    pts = O.ref_random_points(n, 6, 99 + n)
    assert np.array_equal(O.evaluate("d", S, pts).view(np.uint64), O.ref_evaluate(S, pts).view(np.uint64))


@needs_ref
def test_oracle_multithreaded_equals_single_thread():
    S = O.ref_random_system(16, 8, 5, 4, 21)
    pts = O.ref_random_points(16, 37, 22)
    a = O.evaluate("d", S, pts, threads=1)
    b = O.evaluate("d", S, pts, threads=5)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@needs_ref
def test_oracle_mult_tally_matches_closed_form():
    # ref tests/test_engine.cpp:145-158
    n, m, k, d = 8, 5, 4, 6
    S = O.ref_random_system(n, m, k, d, 17)
    pts = O.ref_random_points(n, 25, 18)
    _, cnt = O.evaluate("d", S, pts, counts=True)
    assert cnt["powers"] == n * (d - 2) * 25
    assert cnt["factors"] == n * m * (k - 1) * 25
    assert cnt["stage2"] == n * m * (5 * k - 4) * 25
    assert cnt["speelpenning"] == n * m * (3 * k - 6) * 25


# ---- ref tests/test_kernels.cpp known answers, restated (d and dd)
def _c(vals, W):
    a = np.zeros((len(vals), W))
    for i, v in enumerate(vals):
        a[i, 0] = v.real
        a[i, 2 if W == 4 else 1] = v.imag
    return a


@pytest.mark.parametrize("prec,W", [("d", 2), ("dd", 4)])
def test_speelpenning_2_3_5(prec, W):
    L, mults = O.speelpenning(prec, _c([2, 3, 5], W))
    assert [L[j, 0] for j in range(3)] == [15, 10, 6]
    assert mults == 3


@pytest.mark.parametrize("prec,W", [("d", 2), ("dd", 4)])
@pytest.mark.parametrize("k", [1, 2, 3, 7, 16])
def test_speelpenning_all_ones(prec, W, k):
    L, _ = O.speelpenning(prec, _c([1] * k, W))
    assert np.all(L[:, 0] == 1) and np.all(L[:, 1:] == 0)


def test_speelpenning_small_k():
    L, m = O.speelpenning("d", _c([7 - 2j], 2))
    assert list(L[0]) == [1, 0] and m == 0
    L, m = O.speelpenning("d", _c([7 - 2j, 4 + 1j], 2))
    assert list(L[0]) == [4, 1] and list(L[1]) == [7, -2] and m == 0


@needs_ref
@pytest.mark.parametrize("k", range(1, 21))
def test_speelpenning_brute_force_and_budget(k):
    # ref tests/test_kernels.cpp:118-142 (1e-12 in double) + dd against exact products
    import mpmath as mp
    mp.mp.prec = 250
    pts = O.ref_random_points(k, 1, k)[0]
    z = pts[:, 0] + 1j * pts[:, 1]
    L, mults = O.speelpenning("d", np.ascontiguousarray(pts))
    for j in range(k):
        want = np.prod(np.delete(z, j)) if k > 1 else 1.0
        got = L[j, 0] + 1j * L[j, 1]
        assert abs(got - want) <= 1e-12 * max(abs(got), abs(want), 1e-300)
    assert mults == (3 * k - 6 if k >= 3 else 0)
    Ldd, _ = O.speelpenning("dd", _c(z, 4))
    for j in range(k):
        want = mp.mpc(1)
        for r in range(k):
            if r != j:
                want *= mp.mpc(z[r].real, z[r].imag)
        got = mp.mpc(mp.mpf(Ldd[j, 0]) + mp.mpf(Ldd[j, 1]), mp.mpf(Ldd[j, 2]) + mp.mpf(Ldd[j, 3]))
        assert abs(got - want) <= 1e-30 * max(abs(want), 1e-300) * k


def _single_monomial(coeff, pos, exps, d):
    k = len(pos)
    return dict(n=3, m=1, k=k, d=d, pos=np.array(pos * 3, np.int32), exps=np.array(exps * 3, np.int32),
                coeffs=np.tile(np.array([coeff.real, 0.0, coeff.imag, 0.0]), (3, 1)))


@pytest.mark.parametrize("prec,W", [("d", 2), ("dd", 4)])
def test_stage2_pure_product(prec, W):
    # ref tests/test_kernels.cpp:155-175: 1*x1*x2*x3 at (2,3,5): dx = (15,10,6), value 30
    S = _single_monomial(1 + 0j, [0, 1, 2], [1, 1, 1], 1)
    out = O.evaluate(prec, S, _c([2, 3, 5], W)[None])[0]
    assert out[0, 0] == 30 and [out[3 + i, 0] for i in range(3)] == [15, 10, 6]


@pytest.mark.parametrize("prec,W", [("d", 2), ("dd", 4)])
def test_stage2_prescaled_coefficients(prec, W):
    # ref tests/test_kernels.cpp:177-196: 3*x1^3 x2^7 x3^2 at ones: (9, 21, 6), value 3
    S = _single_monomial(3 + 0j, [0, 1, 2], [3, 7, 2], 7)
    out = O.evaluate(prec, S, _c([1, 1, 1], W)[None])[0]
    assert out[0, 0] == 3 and [out[3 + i, 0] for i in range(3)] == [9, 21, 6]


@pytest.mark.parametrize("prec,W", [("d", 2), ("dd", 4)])
def test_identity_and_duplicate_supports(prec, W):
    # ref tests/test_engine.cpp:62-68 and :181-196
    S = dict(n=1, m=1, k=1, d=1, pos=np.array([0], np.int32), exps=np.array([1], np.int32),
             coeffs=np.array([[1.0, 0, 0, 0]]))
    out = O.evaluate(prec, S, _c([4], W)[None])[0]
    assert out[0, 0] == 4 and out[1, 0] == 1
    S = dict(n=2, m=2, k=2, d=1, pos=np.array([0, 1] * 4, np.int32), exps=np.array([1, 1] * 4, np.int32),
             coeffs=np.tile([0.5, 0, 0, 0], (4, 1)).astype(np.float64))
    out = O.evaluate(prec, S, _c([3, 5], W)[None])[0]
    assert out[0, 0] == 15 and out[2, 0] == 5 and out[3, 0] == 3


# ---- ref tests/test_packing.cpp: slot map and mask
def test_mons_slot_known_answers():
    assert O.mons_slot(0, "value", -1, 32, 32) == 0
    assert O.mons_slot(0, "deriv", 0, 32, 32) == 32
    assert O.mons_slot(33, "value", -1, 32, 32) == 1057
    assert O.mons_slot(1024, "value", -1, 32, 32) == -1
    assert O.mons_slot(0, "deriv", 32, 32, 32) == -1


@needs_ref
@pytest.mark.parametrize("shape", [(4, 1, 1, 1), (4, 4, 2, 3), (8, 3, 8, 2), (16, 16, 9, 2), (32, 32, 9, 2)])
def test_oracle_zero_mask_equals_reference(shape):
    S = O.ref_random_system(*shape, 500 + shape[0])
    assert np.array_equal(O.zero_mask(S), O.ref_zero_mask(S))


@needs_ref
def test_zero_mask_size():
    S = O.ref_random_system(32, 32, 9, 2, 3)
    assert len(O.zero_mask(S)) == 33792 - 10240


# ---- dd primitives against exact arithmetic
def test_cdd_mul_add_error_bounds():
    import mpmath as mp
    mp.mp.prec = 250
    rng = np.random.default_rng(5)
    worst_m = worst_a = 0.0
    for _ in range(2000):
        a = np.zeros(4)
        b = np.zeros(4)
        for v in (a, b):
            v[0], v[2] = rng.uniform(-1, 1, 2) * 2.0 ** rng.integers(-20, 20, 2)
            v[1], v[3] = v[0] * 2.0 ** -54 * rng.uniform(-1, 1), v[2] * 2.0 ** -54 * rng.uniform(-1, 1)
        A = mp.mpc(mp.mpf(a[0]) + mp.mpf(a[1]), mp.mpf(a[2]) + mp.mpf(a[3]))
        Bm = mp.mpc(mp.mpf(b[0]) + mp.mpf(b[1]), mp.mpf(b[2]) + mp.mpf(b[3]))
        r = O.cdd_mul(a, b)
        R = mp.mpc(mp.mpf(r[0]) + mp.mpf(r[1]), mp.mpf(r[2]) + mp.mpf(r[3]))
        worst_m = max(worst_m, float(abs(R - A * Bm) / (abs(A) * abs(Bm))))
        r = O.cdd_add(a, b)
        R = mp.mpc(mp.mpf(r[0]) + mp.mpf(r[1]), mp.mpf(r[2]) + mp.mpf(r[3]))
        worst_a = max(worst_a, float(abs(R - (A + Bm)) / (abs(A) + abs(Bm))))
    # normwise bounds: a few u^2 (u^2 = 2^-106 = 1.23e-32)
    assert worst_m < 8 * 2.0 ** -106, worst_m
    assert worst_a < 4 * 2.0 ** -106, worst_a

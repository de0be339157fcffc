"""Wide encoding: n > 256 behind PJ_CTX_WIDE.

The reference rejects n > 256 (build_layout, ref src/packing.cpp:25-27); without the option the
B200 library keeps that rejection (same message class, std::invalid_argument -> ValueError).
With it, positions/exponents are packed in 32-bit words and the generic kernel evaluates every
precision and order under the same contracts as the byte encoding:
  * the oracle (any n) is pinned to mpmath on tests/golden/wide (dd, 1e-30 * sum|terms|);
  * host index maps (slot targets, zero mask) equal the oracle's restatement;
  * on the GPU: complex double and dd reference order bit-exact with the oracle, dd fast order
    within 1e-30 * sum|terms| of the mpmath truth and the oracle.
"""
import glob
import os

import numpy as np
import pytest

import paper_1201_0499_b200 as pj
from conftest import DD_TOL, GOLDEN, dd_rel, load_golden, sysd_of
from oracle import oracle as O

WIDE_GOLDEN = sorted(glob.glob(os.path.join(GOLDEN, "wide", "*.npz")))


def system_of(S):
    return pj.PolynomialSystem(S["n"], S["m"], S["k"], S["d"], S["pos"].reshape(-1, S["k"]),
                               S["exps"].reshape(-1, S["k"]), S["coeffs"])


@pytest.mark.parametrize("path", WIDE_GOLDEN, ids=lambda p: p.split("/")[-1])
def test_oracle_dd_matches_mpmath_wide(path):
    S, z = load_golden(path)
    got = O.evaluate("dd", S, z["points_dd"])
    assert dd_rel(got, z["truth_dd"], z["magsum"]) <= DD_TOL


def test_default_context_keeps_the_reference_cap():
    s = pj.random_system(300, 2, 3, 3, 5)
    with pytest.raises(ValueError, match="n > 256"):
        pj.EvaluationContext(s, device=-1)
    pj.EvaluationContext(s, device=-1, wide=True)  # accepted with the option


def test_wide_index_maps_host_only():
    s = pj.random_system(300, 3, 4, 3, 9)
    S = sysd_of(s)
    ctx = pj.EvaluationContext(s, device=-1, wide=True)
    assert np.array_equal(ctx.zero_mask(), O.zero_mask(S))
    n, m = 300, 3
    for sidx in [0, 1, 450, n * m - 1]:
        want = [O.mons_slot(sidx, "derivative", int(v), n, m) for v in S["pos"][sidx * 4:(sidx + 1) * 4]]
        want.append(O.mons_slot(sidx, "value", -1, n, m))
        assert list(ctx.slot_targets(sidx)) == want


def test_wide_limits():
    # k above the 16-bit stage-3 entry range is rejected
    n = 2047
    co = np.zeros((n, 4))
    co[:, 0] = 1.0
    pos = np.tile(np.arange(n, dtype=np.int32), (n, 1))
    s = pj.PolynomialSystem(n, 1, n, 1, pos, np.ones((n, n), np.int32), co)
    with pytest.raises(ValueError, match="k exceeds the wide encoding"):
        pj.EvaluationContext(s, device=-1, wide=True)


@pytest.mark.gpu
@pytest.mark.parametrize("path", WIDE_GOLDEN, ids=lambda p: p.split("/")[-1])
def test_wide_golden_on_device(path, gpu):
    S, z = load_golden(path)
    ctx = pj.EvaluationContext(system_of(S), wide=True)
    want = O.evaluate("dd", S, z["points_dd"])
    got_ref = ctx.evaluate_dd(z["points_dd"], order="ref")
    assert np.array_equal(got_ref, want)
    got = ctx.evaluate_dd(z["points_dd"])
    assert dd_rel(got, z["truth_dd"], z["magsum"]) <= DD_TOL
    p2 = np.ascontiguousarray(z["points_dd"][..., [0, 2]])
    got_d = ctx.evaluate_host(p2, "d")
    assert np.array_equal(got_d.view(np.uint64), O.evaluate("d", S, p2).view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(257, 1, 1, 1, 4), (300, 3, 4, 3, 3), (400, 40, 6, 2, 2), (260, 2, 260, 2, 2)],
                         ids=lambda s: "n%d_m%d_k%d_d%d_B%d" % s)
def test_wide_random_on_device(shape, gpu):
    n, m, k, d, B = shape
    s = pj.random_system(n, m, k, d, 31 + n)
    S = sysd_of(s)
    ctx = pj.EvaluationContext(s, wide=True)
    pts = pj.random_points(n, B, 7)
    p2 = np.stack([pts.real, pts.imag], -1)
    assert np.array_equal(ctx.evaluate_host(p2, "d").view(np.uint64), O.evaluate("d", S, p2).view(np.uint64))
    p4 = pj.to_dd(pts)
    p4[..., 1] = p4[..., 0] * 2.0 ** -55
    want, ms = O.evaluate("dd", S, p4, magsum=True)
    assert np.array_equal(ctx.evaluate_dd(p4, order="ref"), want)
    assert dd_rel(ctx.evaluate_dd(p4), want, ms) <= DD_TOL
    with pytest.raises(ValueError, match="n > 256"):
        ctx.newton_host(p4, "dd")

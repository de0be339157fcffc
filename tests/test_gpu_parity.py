"""Parity of the sm_100a path against the oracle, through the C ABI (needs a B200).

Bars:
  * complex double: bit-exact with the UNMODIFIED reference (oracle/_ref, or the committed
    reference outputs in tests/golden) — same operation order, ascending-g stage-3 sums;
  * complex dd, reference order (PJ_ORDER_REF): bit-equal to the oracle's dd restatement;
  * complex dd, fast order (default): |got - want| <= 1e-30 * sum|terms| against the mpmath
    truth and against the oracle;
  * structural zeros: exact +0 in every word, index maps bit-exact (tests/test_host.py).
"""
import numpy as np
import pytest

import paper_1201_0499_b200 as pj
from conftest import DD_TOL, dd_err, dd_rel, golden_cases, load_golden, sysd_of
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def ctx_of(S, device=0):
    s = pj.PolynomialSystem(S["n"], S["m"], S["k"], S["d"], S["pos"].reshape(-1, S["k"]),
                            S["exps"].reshape(-1, S["k"]), S["coeffs"])
    return pj.EvaluationContext(s, device=device)


def ref_double(S, p2):
    return O.ref_evaluate(S, p2) if O.ref_available() else O.evaluate("d", S, p2)


def stress_dd(pts_c, seed=0):
    p4 = pj.to_dd(pts_c)
    rng = np.random.default_rng(seed)
    p4[..., 1] = p4[..., 0] * 2.0 ** -54 * rng.uniform(-1, 1, p4[..., 0].shape)
    p4[..., 3] = p4[..., 2] * 2.0 ** -54 * rng.uniform(-1, 1, p4[..., 2].shape)
    return p4


@pytest.mark.parametrize("path", golden_cases(), ids=lambda p: p.split("/")[-1])
def test_golden(path, gpu):
    S, z = load_golden(path)
    ctx = ctx_of(S)
    got_d = ctx.evaluate_host(z["points_d"], "d")
    assert np.array_equal(got_d.view(np.uint64), z["ref_d"].view(np.uint64)), "complex double not bit-exact"
    want = O.evaluate("dd", S, z["points_dd"])
    got_ref = ctx.evaluate_dd(z["points_dd"], order="ref")
    assert np.array_equal(got_ref, want), "dd reference order differs from the oracle"
    got = ctx.evaluate_dd(z["points_dd"])
    assert dd_rel(got, z["truth_dd"], z["magsum"]) <= DD_TOL
    assert dd_rel(got_ref, z["truth_dd"], z["magsum"]) <= DD_TOL
    zero = z["magsum"] == 0
    assert np.all(got[zero].view(np.uint64) == 0) and np.all(got_d[zero].view(np.uint64) == 0)


SHAPES = [(32, 32, 9, 2), (32, 32, 16, 10), (8, 3, 3, 5), (4, 4, 1, 1), (32, 32, 8, 2), (64, 64, 16, 10),
          (40, 40, 20, 3), (6, 4, 2, 3), (4, 1, 1, 255), (12, 5, 6, 4), (1, 1, 1, 1), (40, 20, 40, 2),
          (33, 31, 7, 3), (100, 7, 5, 4), (256, 2, 3, 2), (10, 70, 4, 3)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "n%d_m%d_k%d_d%d" % s)
def test_shapes_vs_reference_and_oracle(shape, gpu):
    n, m, k, d = shape
    s = pj.random_system(n, m, k, d, 7000 + n + m + k + d)
    S = sysd_of(s)
    ctx = pj.EvaluationContext(s)
    B = 5 if n * m * k > 20000 else 9
    pts = pj.random_points(n, B, 11 + n)
    p2 = np.stack([pts.real, pts.imag], -1)
    got_d = ctx.evaluate_host(p2, "d")
    assert np.array_equal(got_d.view(np.uint64), ref_double(S, p2).view(np.uint64))
    p4 = stress_dd(pts, n)
    want, ms = O.evaluate("dd", S, p4, magsum=True)
    assert np.array_equal(ctx.evaluate_dd(p4, order="ref"), want)
    assert dd_rel(ctx.evaluate_dd(p4), want, ms) <= DD_TOL


def test_global_scratch_path_huge_table(gpu):
    # n*d too large for shared memory: tables and staging fall back to global scratch
    s = pj.random_system(200, 2, 3, 255, 5)
    ctx = pj.EvaluationContext(s)
    assert ctx.launch("dd")["smem_bytes"] == 0
    S = sysd_of(s)
    pts = pj.random_points(200, 3, 6) * 0.999
    p4 = stress_dd(pts, 1)
    want, ms = O.evaluate("dd", S, p4, magsum=True)
    assert np.array_equal(ctx.evaluate_dd(p4, order="ref"), want)
    assert dd_rel(ctx.evaluate_dd(p4), want, ms) <= DD_TOL
    p2 = np.stack([pts.real, pts.imag], -1)
    assert np.array_equal(ctx.evaluate_host(p2, "d").view(np.uint64), ref_double(S, p2).view(np.uint64))


# ---- the reference's known answers through the GPU path
def _single(coeff, pos, exps, d):
    t = pj.Term(coeff, pj.MonomialSupport(pos, exps))
    return pj.PolynomialSystem.from_terms(3, 1, len(pos), d, [t, t, t])


def test_stage2_known_answers(gpu):
    # ref tests/test_kernels.cpp:155-196
    r = pj.EvaluationContext(_single(1 + 0j, [0, 1, 2], [1, 1, 1], 1)).evaluate([2, 3, 5])
    assert r.values[0] == 30 and [r.jac(0, i) for i in range(3)] == [15, 10, 6]
    r = pj.EvaluationContext(_single(3 + 0j, [0, 1, 2], [3, 7, 2], 7)).evaluate([1, 1, 1])
    assert r.values[0] == 3 and [r.jac(0, i) for i in range(3)] == [9, 21, 6]
    dd = pj.EvaluationContext(_single(3 + 0j, [0, 1, 2], [3, 7, 2], 7)).evaluate_dd(pj.to_dd(np.ones((1, 3))))
    assert dd[0, 0, 0] == 3 and [dd[0, 3 + i, 0] for i in range(3)] == [9, 21, 6]


def test_identity_and_duplicates(gpu):
    # ref tests/test_engine.cpp:62-68, :181-196
    s = pj.PolynomialSystem.from_terms(1, 1, 1, 1, [pj.Term(1, pj.MonomialSupport([0], [1]))])
    r = pj.EvaluationContext(s).evaluate([4])
    assert r.values[0] == 4 and r.jacobian[0] == 1
    t = pj.Term(0.5, pj.MonomialSupport([0, 1], [1, 1]))
    r = pj.EvaluationContext(pj.PolynomialSystem.from_terms(2, 2, 2, 1, [t, t, t, t])).evaluate([3, 5])
    assert r.values[0] == 15 and r.jac(0, 0) == 5 and r.jac(0, 1) == 3


def test_structural_zeros_exact(gpu):
    # ref tests/test_kernels.cpp:301-319
    s = pj.random_system(12, 3, 4, 2, 21)
    r = pj.EvaluationContext(s).evaluate(pj.random_point(12, 22))
    for p in range(12):
        present = set(s.positions[p * 3:(p + 1) * 3].reshape(-1).tolist())
        for i in range(12):
            if i not in present:
                z = np.array([r.jac(p, i)]).view(np.uint64)
                assert np.all(z == 0)


def test_bit_identical_across_launch_shapes(gpu):
    # the analogue of ref tests/test_engine.cpp:85-100 (workers x block sizes)
    s = pj.random_system(32, 22, 9, 2, 1234)
    ctx = pj.EvaluationContext(s)
    pts = stress_dd(pj.random_points(32, 37, 1235), 3)
    base = ctx.evaluate_dd(pts)
    base_d = ctx.evaluate_host(np.stack([pts[..., 0], pts[..., 2]], -1), "d")
    for threads in (32, 64, 128, 256):
        for tp in (1, 2, 3, 8):
            ctx.set_launch("dd", threads, tp)
            ctx.set_launch("d", threads, tp)
            assert np.array_equal(ctx.evaluate_dd(pts).view(np.uint64), base.view(np.uint64))
            got_d = ctx.evaluate_host(np.stack([pts[..., 0], pts[..., 2]], -1), "d")
            assert np.array_equal(got_d.view(np.uint64), base_d.view(np.uint64))


def test_point_validation(gpu):
    # ref tests/test_engine.cpp:298-305
    ctx = pj.EvaluationContext(pj.random_system(4, 2, 2, 2, 8))
    with pytest.raises(ValueError):
        ctx.evaluate(np.ones(3))
    bad = np.ones(4, np.complex128)
    bad[2] = complex(1, np.nan)
    with pytest.raises(ValueError):
        ctx.evaluate(bad)
    p4 = pj.to_dd(np.ones((3, 4)))
    p4[1, 2, 1] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        ctx.evaluate_dd(p4)
    assert ctx.evaluate_dd(pj.to_dd(np.ones((2, 4)))).shape == (2, 20, 4)  # flag cleared


def test_batch_repeat_and_tally(gpu):
    # ref tests/test_engine.cpp:307-345
    ctx = pj.EvaluationContext(pj.random_system(8, 8, 3, 2, 99))
    pt = pj.random_point(8, 98)
    once = ctx.evaluate_batch([pt, pt], 1)
    assert np.array_equal(once.results[0].values, once.results[1].values)
    twice = ctx.evaluate_batch([pt], 2)
    assert np.array_equal(twice.results[0].jacobian, once.results[0].jacobian) and twice.report.evals == 2
    with pytest.raises(ValueError):
        ctx.evaluate_batch([pt], 0)
    empty = ctx.evaluate_batch([], 3)
    assert empty.results == [] and empty.report.evals == 0 and empty.report.mults.total() == 0
    n, m, k, d = 8, 5, 4, 6
    c2 = pj.EvaluationContext(pj.random_system(n, m, k, d, 17))
    rep = c2.evaluate_batch([pj.random_point(n, 18)], 25).report
    assert rep.mults.total() == (n * (d - 2) + n * m * (k - 1) + n * m * (5 * k - 4)) * 25


def test_engine_matches_oracle_at_1e10(gpu):
    # ref tests/test_engine.cpp:70-83 via the naive oracle of the reference (1e-10 gate)
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    for shape in [(32, 32, 9, 2), (32, 32, 16, 10), (8, 3, 3, 5), (4, 4, 1, 1)]:
        s = pj.random_system(*shape, 7000)
        S = sysd_of(s)
        ctx = pj.EvaluationContext(s)
        for t in range(3):
            pt = pj.random_point(shape[0], 7001 + t)
            r = ctx.evaluate(pt)
            want = O.ref_naive(S, np.stack([pt.real, pt.imag], -1))
            w = want[:, 0] + 1j * want[:, 1]
            got = np.concatenate([r.values, r.jacobian])
            den = np.maximum(np.maximum(abs(got), abs(w)), 1e-300)
            rel = np.where((abs(got) < 1e-300) & (abs(w) < 1e-300), abs(got - w), abs(got - w) / den)
            assert rel.max() <= 1e-10


# ---- full-size configurations (size-independent properties + sampled oracle checks)
def _device_run(ctx, p4_host, prec="dd", order=None):
    import torch
    pts = torch.from_numpy(p4_host).cuda()
    W = p4_host.shape[-1]
    out = torch.empty((pts.shape[0], ctx.n + ctx.n * ctx.n, W), dtype=torch.float64, device="cuda")
    ctx.evaluate_device(pts, out, prec, order)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("shape", [(32, 32, 8, 2), (64, 64, 16, 10)], ids=["C2", "C3"])
def test_full_batch_65536(shape, gpu):
    n, m, k, d = shape
    s = pj.random_system(n, m, k, d, 7)
    S = sysd_of(s)
    ctx = pj.EvaluationContext(s)
    B = 65536
    pts = pj.random_points(n, B, 11)
    p4 = pj.to_dd(pts)
    out = _device_run(ctx, p4)
    out2 = _device_run(ctx, p4)
    assert np.array_equal(out.view(np.uint64), out2.view(np.uint64)), "not deterministic"
    assert np.all(np.isfinite(out))
    # structural zeros: Jacobian (p, v) with v absent from row p is +0 for every point
    present = np.zeros((n, n), bool)
    for sidx in range(n * m):
        present[sidx // m, s.positions[sidx]] = True
    jac = out[:, n:, :].reshape(B, n, n, 4)
    assert np.all(jac[:, ~present].view(np.uint64) == 0)
    assert np.all(np.any(jac[:, present] != 0, axis=-1).mean(axis=0) > 0.99)
    # sampled oracle checks (first, last, and random points)
    idx = np.unique(np.concatenate([[0, B - 1], np.random.default_rng(1).integers(0, B, 14)]))
    want, ms = O.evaluate("dd", S, p4[idx], magsum=True, threads=8)
    assert dd_rel(out[idx], want, ms) <= DD_TOL
    # complex double at full size: bit-exact on the sample
    p2 = np.ascontiguousarray(p4[..., [0, 2]])
    outd = _device_run(ctx, p2, "d")
    assert np.array_equal(outd[idx].view(np.uint64), ref_double(S, p2[idx]).view(np.uint64))


def test_host_pipeline_many_chunks_matches_device_path(gpu):
    s = pj.random_system(32, 32, 8, 2, 7)
    ctx = pj.EvaluationContext(s)
    B = 50000
    p4 = pj.to_dd(pj.random_points(32, B, 3))
    dev = _device_run(ctx, p4)
    host = ctx.evaluate_dd(p4)
    assert np.array_equal(dev.view(np.uint64), host.view(np.uint64))


def test_reference_order_dd_full_batch_sample(gpu):
    s = pj.random_system(32, 32, 8, 2, 7)
    S = sysd_of(s)
    ctx = pj.EvaluationContext(s)
    p4 = stress_dd(pj.random_points(32, 4096, 11), 9)
    out = _device_run(ctx, p4, "dd", "ref")
    idx = np.arange(0, 4096, 97)
    assert np.array_equal(out[idx], O.evaluate("dd", S, p4[idx], threads=8))


# ---- the specialised fast kernel (eval_fast.cu): every instantiated k, chunking, strides
@pytest.mark.parametrize("k", list(range(2, 18)))
def test_fast_kernel_each_k(k, gpu):
    n = max(k + 3, 20)
    s = pj.random_system(n, 40, k, 3, 900 + k)   # m = 40: two 32-monomial chunks, one partial
    S = sysd_of(s)
    ctx = pj.EvaluationContext(s)
    want_variant = 1 if 2 <= k <= 16 else -1
    assert ctx.launch("dd")["variant"] == want_variant
    p4 = stress_dd(pj.random_points(n, 7, 901 + k), k)
    want, ms = O.evaluate("dd", S, p4, magsum=True)
    assert dd_rel(ctx.evaluate_dd(p4), want, ms) <= DD_TOL
    ctx.set_variant(-1)  # the generic kernel in the same (fast) order family
    assert dd_rel(ctx.evaluate_dd(p4), want, ms) <= DD_TOL


@pytest.mark.parametrize("shape", [(256, 2, 16, 2), (64, 70, 16, 10), (33, 32, 8, 2), (100, 33, 12, 5)],
                         ids=lambda s: "n%d_m%d_k%d_d%d" % s)
def test_fast_kernel_strides_and_chunks(shape, gpu):
    n, m, k, d = shape
    s = pj.random_system(n, m, k, d, 77)
    S = sysd_of(s)
    ctx = pj.EvaluationContext(s)
    p4 = stress_dd(pj.random_points(n, 4, 78), 2)
    want, ms = O.evaluate("dd", S, p4, magsum=True)
    assert dd_rel(ctx.evaluate_dd(p4), want, ms) <= DD_TOL


def test_fast_kernel_launch_shape_invariance(gpu):
    s = pj.random_system(32, 32, 8, 2, 5)
    ctx = pj.EvaluationContext(s)
    p4 = stress_dd(pj.random_points(32, 29, 6), 4)
    base = ctx.evaluate_dd(p4)
    for threads in (32, 64, 128, 256):
        for tp in (1, 2, 3, 4):
            ctx.set_launch("dd", threads, tp)
            assert np.array_equal(ctx.evaluate_dd(p4).view(np.uint64), base.view(np.uint64))


def test_fast_kernel_wide_ctas_for_large_k(gpu):
    # k > 12: CTAs of up to 16 warps (one SM-filling CTA when the staging dominates shared memory)
    s = pj.random_system(24, 20, 16, 3, 77)
    S = sysd_of(s)
    ctx = pj.EvaluationContext(s)
    p4 = stress_dd(pj.random_points(24, 41, 78), 5)
    want, ms = O.evaluate("dd", S, p4, magsum=True)
    base = ctx.evaluate_dd(p4)
    assert dd_rel(base, want, ms) <= DD_TOL
    for threads in (256, 320, 384):  # 16 warps of staging would exceed shared memory at k = 16
        for tp in (1, 2):
            ctx.set_launch("dd", threads, tp)
            assert ctx.launch("dd")["variant"] == 1
            assert np.array_equal(ctx.evaluate_dd(p4).view(np.uint64), base.view(np.uint64))


def test_concurrent_planning_and_launches_of_mixed_shapes(gpu):
    # contexts of different shapes planned and launched from several threads at once: the
    # kernels' dynamic shared-memory attribute is process-wide, so no context may leave it below
    # another's launch (regression: "too many resources requested for launch" under threads)
    import threading
    shapes = [(32, 32, 8, 2, 41), (24, 20, 16, 3, 42), (40, 45, 5, 4, 43), (32, 32, 8, 2, 44)]
    systems = [pj.random_system(*sh) for sh in shapes]
    pts = [pj.to_dd(pj.random_points(s.n, 67, 50 + i)) for i, s in enumerate(systems)]
    want = [pj.EvaluationContext(s).evaluate_dd(p) for s, p in zip(systems, pts)]
    pts_d = [np.stack([z.real, z.imag], -1).copy() for z in (pj.random_points(s.n, 33, 60 + i) for i, s in enumerate(systems))]
    want_d = [pj.EvaluationContext(s).evaluate_host(p, "d") for s, p in zip(systems, pts_d)]
    errors = []
    barrier = threading.Barrier(len(systems))

    def work(i):
        try:
            barrier.wait()
            ctx = pj.EvaluationContext(systems[i])
            for _ in range(6):
                assert np.array_equal(ctx.evaluate_dd(pts[i]).view(np.uint64), want[i].view(np.uint64))
                got_d = ctx.evaluate_host(pts_d[i], "d")
                assert np.array_equal(got_d.view(np.uint64), want_d[i].view(np.uint64))
        except Exception as exc:  # surfaced below
            errors.append(exc)

    th = [threading.Thread(target=work, args=(i,)) for i in range(len(systems))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors


def test_set_launch_refuses_unrunnable_wide_ctas(gpu):
    # CTAs above 256 threads exist only for the fast dd kernel at k > 12; anything else is
    # refused up front and the previous launch shape is kept (no failing launch later)
    s = pj.random_system(32, 32, 8, 2, 7)
    ctx = pj.EvaluationContext(s)
    before = ctx.launch("dd")
    with pytest.raises(ValueError, match="threads > 256"):
        ctx.set_launch("dd", 384, 1)
    assert ctx.launch("dd") == before
    p4 = pj.to_dd(pj.random_points(32, 5, 3))
    S = sysd_of(s)
    want, ms = O.evaluate("dd", S, p4, magsum=True)
    assert dd_rel(ctx.evaluate_dd(p4), want, ms) <= DD_TOL
    s16 = pj.random_system(64, 64, 16, 10, 7)  # k = 16, n = 64: 12 warps of staging do not fit
    c16 = pj.EvaluationContext(s16)
    with pytest.raises(ValueError, match="threads > 256"):
        c16.set_launch("dd", 384, 1)


def test_dd_contract_under_cancellation(gpu):
    """Adversarial inputs: duplicated monomials with opposite coefficients (exact cancellation
    in every stage-3 sum), unit-modulus points (no decay along k = 16 product chains, d = 10),
    and a wide dynamic range of coordinates."""
    n, m, k, d = 24, 16, 16, 10
    base = pj.random_system(n, m, k, d, 31)
    s = pj.PolynomialSystem(n, m, k, d, base.positions.copy(), base.exponents.copy(), base.coeffs.copy())
    for p in range(n):                      # monomial 2i+1 = monomial 2i with coefficient * -1
        for g in range(0, m, 2):
            a, b = p * m + g, p * m + g + 1
            s.positions[b] = s.positions[a]
            s.exponents[b] = s.exponents[a]
            s.coeffs[b] = -s.coeffs[a]
    S = sysd_of(s)
    ctx = pj.EvaluationContext(s)
    ang = np.random.default_rng(3).uniform(0, 2 * np.pi, (6, n))
    unit = np.exp(1j * ang)
    scale = 2.0 ** np.random.default_rng(4).integers(-12, 12, (6, n))
    for pts in (unit, unit * scale):
        p4 = stress_dd(pts, 5)
        want, ms = O.evaluate("dd", S, p4, magsum=True)
        got = ctx.evaluate_dd(p4)
        assert dd_rel(got, want, ms) <= DD_TOL
        # exact cancellation: every value and Jacobian entry is (near) zero relative to its terms
        mag = np.abs(got[..., 0]) + np.abs(got[..., 2])
        assert np.all(mag <= 1e-30 * np.maximum(ms, 1e-300) + (ms == 0))
    # and a generic system on unit-modulus points (longest undamped chains)
    s2 = pj.random_system(n, m, k, d, 32)
    S2 = sysd_of(s2)
    c2 = pj.EvaluationContext(s2)
    p4 = stress_dd(unit, 6)
    want, ms = O.evaluate("dd", S2, p4, magsum=True)
    assert dd_rel(c2.evaluate_dd(p4), want, ms) <= DD_TOL


def test_distinct_contexts_are_thread_safe(gpu):
    # ref engine.hpp:84-86: one context per thread; distinct contexts may run concurrently
    import threading
    systems = [pj.random_system(32, 32, 8, 2, 900 + i) for i in range(3)]
    pts = [stress_dd(pj.random_points(32, 257, 910 + i), i) for i in range(3)]
    want = [pj.EvaluationContext(s).evaluate_dd(p) for s, p in zip(systems, pts)]
    want_x = [pj.EvaluationContext(s).newton_host(p, "dd")[0] for s, p in zip(systems, pts)]
    errors = []

    def work(i):
        try:
            ctx = pj.EvaluationContext(systems[i])
            for _ in range(4):
                assert np.array_equal(ctx.evaluate_dd(pts[i]).view(np.uint64), want[i].view(np.uint64))
                assert np.array_equal(ctx.newton_host(pts[i], "dd")[0].view(np.uint64), want_x[i].view(np.uint64))
        except Exception as exc:  # surfaced below
            errors.append(exc)

    th = [threading.Thread(target=work, args=(i,)) for i in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("shape", [(32, 32, 8, 2), (64, 64, 16, 10)], ids=["C2", "C3"])
def test_small_batches_split_tiles_bit_identical(shape, gpu):
    """Batches with fewer tiles than CTAs spread each tile's tasks over several CTAs (pj_evaluate,
    eval_fast.cu SP): the arithmetic of a task does not depend on who runs it, so every point's
    results are bit-identical whether it is evaluated alone, in a small batch or in a full one,
    and they stay within the contract of the oracle."""
    n, m, k, d = shape
    s = pj.random_system(n, m, k, d, 7)
    ctx = pj.EvaluationContext(s)
    S = sysd_of(s)
    B = 2000
    p4 = stress_dd(pj.random_points(n, B, 5), seed=3)
    full = ctx.evaluate_dd(p4)
    for b in [1, 2, 3, 7, 100]:
        got = ctx.evaluate_dd(p4[:b])
        assert np.array_equal(got.view(np.uint64), full[:b].view(np.uint64)), b
    got1 = ctx.evaluate_dd(p4[B - 1:])
    assert np.array_equal(got1.view(np.uint64), full[B - 1:].view(np.uint64))
    want, ms = O.evaluate("dd", S, p4[:7], magsum=True)
    assert dd_rel(full[:7], want, ms) <= DD_TOL
    # complex double (its split runs a separate kernel instantiation): bit-exact with the
    # reference at every batch size
    p2 = np.ascontiguousarray(p4[..., [0, 2]])
    full_d = ctx.evaluate_host(p2, "d")
    for b in [1, 2, 3, 7, 100]:
        assert np.array_equal(ctx.evaluate_host(p2[:b], "d").view(np.uint64), full_d[:b].view(np.uint64)), b
    assert np.array_equal(full_d[:3].view(np.uint64), ref_double(S, p2[:3]).view(np.uint64))

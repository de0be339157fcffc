"""Parity of the device Newton corrector (csrc/newton.cu) through the C ABI.

Bars:
  * the solver alone (pj_newton_solve on given evaluator output): bit-exact with the oracle's
    restatement (same operation order), complex double and complex dd, with and without a
    target, shared-memory (n <= 64) and global-slab (n > 64) matrices;
  * evaluate + solve (pj_newton_step / pj_newton_host): bit-exact with the oracle in complex
    double and in dd reference order; the default dd fast order within the mpmath bound;
  * against exact arithmetic (tests/golden/newton): normwise forward error <= n cond(J) u;
  * known answers (permutation system -> exact root, singular J -> status 1), quadratic
    convergence to a known root on the GPU, in-place update (points_out aliasing points).
"""
import glob
import os

import numpy as np
import pytest

import paper_1201_0499_b200 as pj
from conftest import GOLDEN, sysd_of
from oracle import oracle as O
from test_newton_oracle import U, fwd_err, permutation_system

pytestmark = pytest.mark.gpu
NEWTON_GOLDEN = sorted(glob.glob(os.path.join(GOLDEN, "newton", "*.npz")))


def torch_dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def solve_gpu(ctx, prec, ev, pts, target=None):
    import torch
    B, n, W = pts.shape
    e, x = torch_dev(ev), torch_dev(pts)
    t = torch_dev(target) if target is not None else None
    out = torch.empty_like(x)
    norms = torch.empty((B, 2), dtype=torch.float64, device="cuda")
    status = torch.empty(B, dtype=torch.int32, device="cuda")
    ctx.newton_solve_device(e, x, out, prec, target=t, norms=norms, status=status)
    torch.cuda.synchronize()
    return out.cpu().numpy(), norms.cpu().numpy(), status.cpu().numpy()


def shaped(n, m, k, d, B, seed=7):
    s = pj.random_system(n, m, k, d, seed)
    S = sysd_of(s)
    pts = pj.random_points(n, B, 11 + n)
    return s, S, pts


SHAPES = [(32, 32, 8, 2, 64), (64, 64, 16, 10, 8), (8, 3, 3, 5, 33), (33, 31, 7, 3, 9), (1, 1, 1, 1, 5),
          (100, 7, 5, 4, 3), (20, 10, 16, 10, 6)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "n%d_m%d_k%d_d%d_B%d" % s)
@pytest.mark.parametrize("prec", ["d", "dd"])
@pytest.mark.parametrize("with_target", [False, True])
def test_solver_bit_exact_vs_oracle(shape, prec, with_target, gpu):
    n, m, k, d, B = shape
    s, S, pts = shaped(n, m, k, d, B)
    ctx = pj.EvaluationContext(s)
    if prec == "d":
        p = np.stack([pts.real, pts.imag], -1)
    else:
        p = pj.to_dd(pts)
        p[..., 1] = p[..., 0] * 2.0 ** -56
        p[..., 3] = p[..., 2] * -(2.0 ** -57)
    ev = O.evaluate(prec, S, p)
    tg = None
    if with_target:
        tg = 0.5 * np.roll(ev[:, :n], 1, axis=0)
    want = O.newton_solve(prec, n, ev, p, target=tg)
    got = solve_gpu(ctx, prec, ev, p, target=tg)
    assert np.array_equal(got[2], want[2])
    assert np.array_equal(got[0].view(np.uint64), want[0].view(np.uint64))
    assert np.array_equal(got[1].view(np.uint64), want[1].view(np.uint64))


@pytest.mark.parametrize("path", NEWTON_GOLDEN, ids=lambda p: p.split("/")[-1])
@pytest.mark.parametrize("prec", ["dd", "d"])
def test_solver_vs_mpmath(path, prec, gpu):
    z = np.load(path)
    n = int(z["n"])
    s = pj.PolynomialSystem(n, int(z["m"]), int(z["k"]), int(z["d"]), z["pos"].reshape(-1, int(z["k"])),
                            z["exps"].reshape(-1, int(z["k"])), z["coeffs"])
    ctx = pj.EvaluationContext(s)
    ev = z["evals_dd"] if prec == "dd" else np.ascontiguousarray(z["evals_dd"][..., [0, 2]])
    B = ev.shape[0]
    dx, norms, status = solve_gpu(ctx, prec, ev, np.zeros((B, n, 4 if prec == "dd" else 2)))
    assert np.all(status == 0)
    assert np.all(fwd_err(dx, z["dx_" + prec], prec) <= n * z["cond"] * U[prec])


@pytest.mark.parametrize("prec,order", [("d", None), ("dd", "ref")])
def test_newton_host_bit_exact_vs_oracle(prec, order, gpu):
    s, S, pts = shaped(32, 32, 8, 2, 300)
    ctx = pj.EvaluationContext(s)
    p = np.stack([pts.real, pts.imag], -1) if prec == "d" else pj.to_dd(pts)
    got, gn, gs = ctx.newton_host(p, prec, iters=3, order=order)
    x = p
    for _ in range(3):
        x, wn, ws = O.newton_solve(prec, 32, O.evaluate(prec, S, x), x)
    assert np.array_equal(gs, ws)
    assert np.array_equal(got.view(np.uint64), x.view(np.uint64))
    assert np.array_equal(gn.view(np.uint64), wn.view(np.uint64))


def test_newton_host_fast_order_converges_to_known_root(gpu):
    s, S, _ = shaped(32, 32, 8, 2, 1)
    xs = pj.to_dd(pj.random_points(32, 256, 21))
    y = O.evaluate("dd", S, xs)[:, :32]
    rng = np.random.default_rng(1)
    x0 = xs.copy()
    x0[..., 0] += 1e-3 * rng.uniform(-1, 1, x0[..., 0].shape)
    x0[..., 2] += 1e-3 * rng.uniform(-1, 1, x0[..., 2].shape)
    ctx = pj.EvaluationContext(s)
    x, norms, status = ctx.newton_host(x0, "dd", iters=7, target=y)
    ok = status == 0
    assert ok.mean() > 0.95  # a few random starts may sit near a singular Jacobian
    err = np.max(np.abs((x[..., 0] - xs[..., 0]) + (x[..., 1] - xs[..., 1])), axis=1)
    err = np.maximum(err, np.max(np.abs((x[..., 2] - xs[..., 2]) + (x[..., 3] - xs[..., 3])), axis=1))
    assert np.median(err[ok]) < 1e-29
    assert np.median(norms[ok, 1]) < 1e-28  # last step at round-off level


@pytest.mark.parametrize("prec", ["d", "dd"])
def test_known_answers_on_device(prec, gpu):
    s = permutation_system(12)
    ctx = pj.EvaluationContext(s)
    pts = pj.random_points(12, 40, 5)
    p = np.stack([pts.real, pts.imag], -1) if prec == "d" else pj.to_dd(pts)
    x, norms, status = ctx.newton_host(p, prec, iters=1)
    assert np.all(status == 0) and np.all(x.view(np.uint64) == 0)
    # singular: variable 3 in no monomial
    pos = np.array([[0], [1], [2], [0], [1], [2], [2], [0]], np.int32)
    co = np.zeros((8, 4))
    co[:, 0] = np.arange(1, 9)
    s2 = pj.PolynomialSystem(4, 2, 1, 2, pos, np.array([[1], [2]] * 4, np.int32), co)
    ctx2 = pj.EvaluationContext(s2)
    W = 2 if prec == "d" else 4
    p2 = np.zeros((3, 4, W))
    p2[..., 0] = 0.25
    x2, n2, st2 = ctx2.newton_host(p2, prec, iters=2)
    assert np.all(st2 == 1) and np.array_equal(x2, p2) and np.all(np.isinf(n2[:, 1]))


def test_step_device_in_place_and_errors(gpu):
    import torch
    s, S, pts = shaped(32, 32, 8, 2, 50)
    ctx = pj.EvaluationContext(s)
    p = pj.to_dd(pts)
    x = torch_dev(p)
    work = torch.empty((50, 32 + 32 * 32, 4), dtype=torch.float64, device="cuda")
    ctx.newton_step_device(x, work, x, "dd", order="ref")  # in place
    torch.cuda.synchronize()
    want, _, _ = O.newton_solve("dd", 32, O.evaluate("dd", S, p), p)
    assert np.array_equal(x.cpu().numpy().view(np.uint64), want.view(np.uint64))
    assert np.array_equal(work.cpu().numpy(), O.evaluate("dd", S, p))  # work holds f, J
    with pytest.raises(ValueError):
        ctx.newton_host(p[:, :31], "dd")
    with pytest.raises(ValueError):
        ctx.newton_host(p, "dd", iters=0)
    bad = p.copy()
    bad[3, 4, 0] = np.nan
    with pytest.raises(ValueError):
        ctx.newton_host(bad, "dd")


def test_step_device_chunked_fork_join(gpu):
    # batches of >= 2 chunks (4 evaluation waves each) run over two internal streams with
    # fork/join events on the caller's stream: same bits as the oracle, in place, on a side stream
    import torch
    s, S, pts = shaped(32, 32, 8, 2, 9000)
    ctx = pj.EvaluationContext(s)
    p = pj.to_dd(pts)
    x = torch_dev(p)
    work = torch.empty((9000, 32 + 32 * 32, 4), dtype=torch.float64, device="cuda")
    st = torch.empty(9000, dtype=torch.int32, device="cuda")
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        ctx.newton_step_device(x, work, x, "dd", order="ref", status=st, stream=side)
        x2 = x.clone()  # ordered after the join on the caller's stream
    side.synchronize()
    want, _, wst = O.newton_solve("dd", 32, O.evaluate("dd", S, p, threads=8), p, threads=8)
    assert np.array_equal(x2.cpu().numpy().view(np.uint64), want.view(np.uint64))
    assert np.array_equal(st.cpu().numpy(), wst)


@pytest.mark.parametrize("prec", ["d", "dd"])
def test_panel_kernel_bit_identical(prec, gpu):
    # the opt-in blocked solve (n <= 32) computes the same bits as the column kernel and the oracle
    for (n, m, k, d, B) in [(32, 32, 8, 2, 70), (30, 12, 5, 3, 9), (13, 4, 3, 4, 11), (5, 3, 2, 2, 4)]:
        s, S, pts = shaped(n, m, k, d, B)
        ctx = pj.EvaluationContext(s)
        ctx.set_variant(1, prec, newton=True)
        assert ctx.launch(prec, newton=True)["variant"] == 1
        p = np.stack([pts.real, pts.imag], -1) if prec == "d" else pj.to_dd(pts)
        ev = O.evaluate(prec, S, p)
        tg = 0.25 * np.roll(ev[:, :n], 1, axis=0)
        want = O.newton_solve(prec, n, ev, p, target=tg)
        got = solve_gpu(ctx, prec, ev, p, target=tg)
        assert np.array_equal(got[2], want[2])
        assert np.array_equal(got[0].view(np.uint64), want[0].view(np.uint64))
    with pytest.raises(ValueError):
        pj.EvaluationContext(pj.random_system(40, 4, 3, 2, 1)).set_variant(1, "dd", newton=True)


# ---- the mixed-precision solve (PJ_NEWTON_MIXED): complex-double factors + dd refinement
MIXED_SHAPES = [(32, 32, 8, 2, 64), (8, 3, 3, 5, 33), (1, 1, 1, 1, 5), (20, 10, 16, 10, 6), (31, 17, 4, 3, 40)]


@pytest.mark.parametrize("shape", MIXED_SHAPES, ids=lambda s: "n%d_m%d_k%d_d%d_B%d" % s)
@pytest.mark.parametrize("with_target", [False, True])
def test_mixed_solver_bit_exact_vs_oracle(shape, with_target, gpu):
    n, m, k, d, B = shape
    s, S, pts = shaped(n, m, k, d, B)
    ctx = pj.EvaluationContext(s)
    p = pj.to_dd(pts)
    p[..., 1] = p[..., 0] * 2.0 ** -56
    ev = O.evaluate("dd", S, p)
    tg = 0.5 * np.roll(ev[:, :n], 1, axis=0) if with_target else None
    want = O.newton_solve("mixed", n, ev, p, target=tg)
    got = solve_gpu(ctx, "mixed", ev, p, target=tg)
    assert np.array_equal(got[2], want[2])
    assert np.array_equal(got[0].view(np.uint64), want[0].view(np.uint64))
    assert np.array_equal(got[1].view(np.uint64), want[1].view(np.uint64))


@pytest.mark.parametrize("path", [p for p in NEWTON_GOLDEN if int(np.load(p)["n"]) <= 32],
                         ids=lambda p: p.split("/")[-1])
def test_mixed_solver_vs_mpmath(path, gpu):
    z = np.load(path)
    n = int(z["n"])
    s = pj.PolynomialSystem(n, int(z["m"]), int(z["k"]), int(z["d"]), z["pos"].reshape(-1, int(z["k"])),
                            z["exps"].reshape(-1, int(z["k"])), z["coeffs"])
    ctx = pj.EvaluationContext(s)
    ev = z["evals_dd"]
    B = ev.shape[0]
    dx, norms, status = solve_gpu(ctx, "mixed", ev, np.zeros((B, n, 4)))
    assert np.all(status == 0)
    assert np.all(fwd_err(dx, z["dx_dd"], "dd") <= 1e-29)


def test_mixed_step_and_host_bit_exact_vs_oracle(gpu):
    import torch
    s, S, pts = shaped(32, 32, 8, 2, 3000)
    ctx = pj.EvaluationContext(s)
    p = pj.to_dd(pts)
    # host path, 2 iterations, dd reference order evaluation (bit-exact with the oracle's)
    got, gn, gs = ctx.newton_host(p[:300], "mixed", iters=2, order="ref")
    x = p[:300]
    for _ in range(2):
        x, wn, ws = O.newton_solve("mixed", 32, O.evaluate("dd", S, x), x)
    assert np.array_equal(gs, ws)
    assert np.array_equal(got.view(np.uint64), x.view(np.uint64))
    # device step (chunked over two streams for a large batch) = solve on the evaluator's output
    xd = torch_dev(p)
    work = torch.empty((3000, 32 + 1024, 4), dtype=torch.float64, device="cuda")
    out = torch.empty_like(xd)
    st = torch.empty(3000, dtype=torch.int32, device="cuda")
    ctx.newton_step_device(xd, work, out, "mixed", status=st, order="ref")
    torch.cuda.synchronize()
    want = O.newton_solve("mixed", 32, O.evaluate("dd", S, p), p)
    assert np.array_equal(st.cpu().numpy(), want[2])
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want[0].view(np.uint64))


def test_mixed_rejects_large_n_and_flags_ill_conditioning(gpu):
    s, S, pts = shaped(33, 31, 7, 3, 2)
    ctx = pj.EvaluationContext(s)
    p = pj.to_dd(pts)
    ev = O.evaluate("dd", S, p)
    with pytest.raises(ValueError, match="n <= 32"):
        solve_gpu(ctx, "mixed", ev, p)
    s, S, pts = shaped(32, 32, 8, 2, 1)
    ctx = pj.EvaluationContext(s)
    p = pj.to_dd(pts)
    ev = O.evaluate("dd", S, p)
    J = ev[0, 32:].reshape(32, 32, 4)
    J[1] = J[0]
    J[1, :, 0] *= 1.0 + 2.0 ** -40
    J[1, :, 1] = 0.0
    J[1, :, 3] = 0.0
    got = solve_gpu(ctx, "mixed", ev, p)
    want = O.newton_solve("mixed", 32, ev, p)
    assert got[2][0] == 3 == want[2][0]
    assert np.array_equal(got[0].view(np.uint64), want[0].view(np.uint64))

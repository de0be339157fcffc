"""Error semantics and buffer contracts of the device API (GPU).

* PJ_VALIDATE rejects a non-finite batch before writing any output (ref src/engine.cpp:183-188);
* a flag left by an asynchronous call does not fail a later host-API call;
* pj_newton_host reports a diverged iterate per point (status 2) instead of failing the batch;
* device-tensor entry points reject wrong dtype / layout / device / shape before any launch;
* chunked host paths over global-scratch systems (tables beyond shared memory) give the same
  bits as one launch (the per-CTA slabs are never shared by concurrent launches).
"""
import numpy as np
import pytest

import paper_1201_0499_b200 as pj

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_validate_rejects_before_writing(torch_cuda):
    torch = torch_cuda
    ctx = pj.EvaluationContext(pj.random_system(6, 4, 3, 3, 5))
    pts = torch.from_numpy(pj.to_dd(pj.random_points(6, 40, 6))).cuda()
    out = torch.full((40, 42, 4), 7.0, dtype=torch.float64, device="cuda")
    pts[17, 3, 2] = float("nan")
    with pytest.raises(ValueError, match="non-finite"):
        ctx.evaluate_device(pts, out, "dd", validate=True)
    torch.cuda.synchronize()
    assert bool((out == 7.0).all())  # nothing written
    # complex double: same contract
    p2 = torch.from_numpy(np.stack([pj.random_points(6, 5, 7).real, pj.random_points(6, 5, 7).imag], -1).copy()).cuda()
    o2 = torch.full((5, 42, 2), 3.0, dtype=torch.float64, device="cuda")
    p2[4, 5, 0] = float("inf")
    with pytest.raises(ValueError, match="non-finite"):
        ctx.evaluate_device(p2, o2, "d", validate=True)
    torch.cuda.synchronize()
    assert bool((o2 == 3.0).all())
    # a finite batch evaluates normally and matches the unvalidated launch bit for bit
    pts[17, 3, 2] = 0.25
    a = torch.empty_like(out)
    ctx.evaluate_device(pts, out, "dd", validate=True)
    ctx.evaluate_device(pts, a, "dd")
    torch.cuda.synchronize()
    assert torch.equal(out, a)


def test_stale_async_flag_does_not_fail_host_call(torch_cuda):
    torch = torch_cuda
    ctx = pj.EvaluationContext(pj.random_system(6, 4, 3, 3, 5))
    pts = torch.from_numpy(pj.to_dd(pj.random_points(6, 4, 6))).cuda()
    pts[0, 0, 0] = float("nan")
    out = torch.empty((4, 42, 4), dtype=torch.float64, device="cuda")
    ctx.evaluate_device(pts, out, "dd")  # flag raised, never polled
    torch.cuda.synchronize()
    good = pj.to_dd(pj.random_points(6, 3, 8))
    assert ctx.evaluate_dd(good).shape == (3, 42, 4)  # no stale PJ_ENONFINITE
    # ... and the asynchronous flag is still reported (and cleared) by its own poll
    ctx.evaluate_device(pts, out, "dd")
    assert ctx.nonfinite_seen() is True
    assert ctx.nonfinite_seen() is False


def test_newton_host_diverged_point_is_per_point_status():
    # f(x) = x^2 (n = m = k = 1, d = 2): from x = 1e200 the residual overflows to inf, the step is
    # non-finite (status 2); the second point converges (x halves per step). The batch succeeds.
    t = [pj.Term(1.0, pj.MonomialSupport([0], [2]))]
    ctx = pj.EvaluationContext(pj.PolynomialSystem.from_terms(1, 1, 1, 2, t))
    x = pj.to_dd(np.array([[1e200], [0.5]]))
    xo, norms, status = ctx.newton_host(x, "dd", iters=1)
    assert status[0] == 2 and status[1] == 0 and xo[1, 0, 0] == 0.25
    # later iterations evaluate the non-finite iterate: still no batch failure (a NaN Jacobian has
    # no admissible pivot, so the point may end singular instead), the other point converges
    xo, norms, status = ctx.newton_host(x, "dd", iters=3)
    assert status[0] in (1, 2) and status[1] == 0
    assert xo[1, 0, 0] == 0.0625
    # a non-finite INPUT is still rejected up front
    x[1, 0, 0] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        ctx.newton_host(x, "dd", iters=1)
    # and the context keeps working
    xo, _, status = ctx.newton_host(pj.to_dd(np.array([[0.5]])), "dd", iters=1)
    assert status[0] == 0 and xo[0, 0, 0] == 0.25


def test_device_tensor_contracts(torch_cuda):
    torch = torch_cuda
    ctx = pj.EvaluationContext(pj.random_system(6, 4, 3, 3, 5))
    ok_p = torch.zeros((4, 6, 4), dtype=torch.float64, device="cuda")
    ok_o = torch.empty((4, 42, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(TypeError):
        ctx.evaluate_device(ok_p.float(), ok_o, "dd")
    with pytest.raises(ValueError, match="contiguous"):
        ctx.evaluate_device(torch.zeros((4, 6, 8), dtype=torch.float64, device="cuda")[..., ::2], ok_o, "dd")
    with pytest.raises(ValueError, match="cuda"):
        ctx.evaluate_device(ok_p.cpu(), ok_o, "dd")
    with pytest.raises(ValueError, match="shape"):
        ctx.evaluate_device(ok_p, ok_o[:3], "dd")
    xo = torch.empty((4, 6, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(TypeError, match="int32"):
        ctx.newton_solve_device(ok_o, ok_p, xo, "dd", status=torch.zeros(4, dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError, match="shape"):
        ctx.newton_solve_device(ok_o, ok_p, xo, "dd", norms=torch.zeros(3, 2, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError, match="shape"):
        ctx.newton_step_device(ok_p, ok_o, xo, "dd", status=torch.zeros(5, dtype=torch.int32, device="cuda"))


def test_chunked_host_path_on_global_scratch_matches_one_launch(torch_cuda):
    # d = 255 power tables for n = 120 exceed shared memory: the generic kernel's global-scratch
    # variant. evaluate_host cuts B = 5000 points into several chunks; they must not overlap.
    torch = torch_cuda
    s = pj.random_system(120, 2, 2, 255, 3)
    ctx = pj.EvaluationContext(s)
    assert ctx.launch("d")["smem_bytes"] == 0  # global scratch in use
    z = pj.random_points(120, 5000, 4) * 0.999
    p2 = np.ascontiguousarray(np.stack([z.real, z.imag], -1))
    host = ctx.evaluate_host(p2, "d")
    dev_in = torch.from_numpy(p2).cuda()
    dev_out = torch.empty((5000, 120 + 120 * 120, 2), dtype=torch.float64, device="cuda")
    ctx.evaluate_device(dev_in, dev_out, "d")
    torch.cuda.synchronize()
    assert np.array_equal(host.view(np.uint64), dev_out.cpu().numpy().view(np.uint64))


def test_newton_chunked_paths_on_global_slabs_match_one_launch(torch_cuda):
    # n = 100 dd: the augmented matrix (100 x 101 complex dd) exceeds shared memory, so the solve
    # runs on per-CTA global slabs. pj_newton_host (several chunks) and pj_newton_step (chunked
    # fork path) must give the bits of one evaluate + one solve launch.
    torch = torch_cuda
    s = pj.random_system(100, 2, 2, 2, 12)
    ctx = pj.EvaluationContext(s)
    assert ctx.launch("dd", newton=True)["variant"] == 2  # global slabs
    B = 8000
    x = pj.to_dd(pj.random_points(100, B, 13))
    xo_host, _, st_host = ctx.newton_host(x, "dd", iters=1)
    xd = torch.from_numpy(x).cuda()
    work = torch.empty((B, 100 + 100 * 100, 4), dtype=torch.float64, device="cuda")
    xo = torch.empty_like(xd)
    st = torch.empty(B, dtype=torch.int32, device="cuda")
    ctx.evaluate_device(xd, work, "dd")
    ctx.newton_solve_device(work, xd, xo, "dd", status=st)
    torch.cuda.synchronize()
    assert np.array_equal(xo_host.view(np.uint64), xo.cpu().numpy().view(np.uint64))
    assert np.array_equal(st_host, st.cpu().numpy())
    xo2 = torch.empty_like(xd)
    ctx.newton_step_device(xd, work, xo2, "dd")
    torch.cuda.synchronize()
    assert torch.equal(xo2, xo)


def test_small_host_batches_graph_replay_semantics(torch_cuda):
    # small host batches replay one cached CUDA graph (csrc/capi.cpp, pj_evaluate_host): a
    # non-finite point is still rejected, the flag does not leak into the next call, and changes
    # of batch size or precision (re-capture) keep the results identical to a fresh context's
    s = pj.random_system(12, 9, 4, 2, 21)
    ctx, fresh = pj.EvaluationContext(s), pj.EvaluationContext(s)
    pts = pj.to_dd(pj.random_points(12, 5, 22))
    bad = pts.copy()
    bad[2, 7, 0] = float("nan")
    first = ctx.evaluate_dd(pts)
    with pytest.raises(ValueError, match="non-finite"):
        ctx.evaluate_dd(bad)
    for _ in range(3):  # replays after the failed call: no stale flag, same bits
        assert np.array_equal(ctx.evaluate_dd(pts).view(np.uint64), first.view(np.uint64))
    p2 = np.ascontiguousarray(pts[..., [0, 2]])
    for b in [1, 5, 2, 5, 1]:  # alternate batch sizes and precisions
        assert np.array_equal(ctx.evaluate_dd(pts[:b]).view(np.uint64), fresh.evaluate_dd(pts[:b]).view(np.uint64))
        assert np.array_equal(ctx.evaluate_host(p2[:b], "d").view(np.uint64),
                              fresh.evaluate_host(p2[:b], "d").view(np.uint64))
    # a launch-shape change invalidates the cached graph
    ctx.set_launch("dd", 128, 1)
    assert np.array_equal(ctx.evaluate_dd(pts).view(np.uint64), first.view(np.uint64))

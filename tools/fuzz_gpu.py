"""Developer: randomized parity sweep on the GPU (not part of the test suite): random shapes,
batch sizes and seeds through every evaluation precision / order and the Newton solves, each
checked against the oracle (bit-exact where the contract is bit-exact, the dd tolerance otherwise).
    python tools/fuzz_gpu.py [cases] [seed]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1201_0499_b200 as pj
from oracle import oracle as O

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)


def sysd(s):
    return dict(n=s.n, m=s.m, k=s.k, d=s.d, pos=np.ascontiguousarray(s.positions, np.int32).reshape(-1),
                exps=np.ascontiguousarray(s.exponents, np.int32).reshape(-1), coeffs=np.ascontiguousarray(s.coeffs))


def dd_rel(got, want, ms):
    err = np.maximum(np.abs((got[..., 0] - want[..., 0]) + (got[..., 1] - want[..., 1])),
                     np.abs((got[..., 2] - want[..., 2]) + (got[..., 3] - want[..., 3])))
    return float(np.max(err / np.maximum(ms, 1e-300)))


worst = 0.0
for c in range(cases):
    n = int(rng.integers(1, 70))
    k = int(rng.integers(1, min(n, 18) + 1))
    m = int(rng.integers(1, 70))
    d = int(rng.choice([1, 2, 2, 3, 5, 10]))
    B = int(rng.choice([1, 2, 3, 7, 33, 100, 700, 2000]))
    seed = int(rng.integers(1, 1 << 30))
    s = pj.random_system(n, m, k, d, seed)
    S = sysd(s)
    ctx = pj.EvaluationContext(s)
    pts = pj.random_points(n, B, seed + 1)
    p2 = np.stack([pts.real, pts.imag], -1)
    p4 = pj.to_dd(pts)
    p4[..., 1] = p4[..., 0] * 2.0 ** -55
    got_d = ctx.evaluate_host(p2, "d")
    want_d = O.ref_evaluate(S, p2) if O.ref_available() else O.evaluate("d", S, p2)
    assert np.array_equal(got_d.view(np.uint64), want_d.view(np.uint64)), ("d", n, m, k, d, B, seed)
    want4, ms = O.evaluate("dd", S, p4, magsum=True)
    got_ref = ctx.evaluate_dd(p4, order="ref")
    assert np.array_equal(got_ref.view(np.uint64), want4.view(np.uint64)), ("dd ref", n, m, k, d, B, seed)
    got_fast = ctx.evaluate_dd(p4)
    e = dd_rel(got_fast, want4, ms)
    worst = max(worst, e)
    assert e <= 1e-30, ("dd fast", n, m, k, d, B, seed, e)
    Bn = min(B, 64)
    for prec, ev, p in [("d", want_d[:Bn], p2[:Bn]), ("dd", want4[:Bn], p4[:Bn])] + \
                       ([("mixed", want4[:Bn], p4[:Bn])] if n <= 32 else []):
        import torch
        e_, x_ = torch.from_numpy(np.ascontiguousarray(ev)).cuda(), torch.from_numpy(np.ascontiguousarray(p)).cuda()
        out = torch.empty_like(x_)
        nr = torch.empty((Bn, 2), dtype=torch.float64, device="cuda")
        st = torch.empty(Bn, dtype=torch.int32, device="cuda")
        ctx.newton_solve_device(e_, x_, out, prec, norms=nr, status=st)
        torch.cuda.synchronize()
        wx, wn, ws = O.newton_solve(prec, n, ev, p)
        assert np.array_equal(st.cpu().numpy(), ws), (prec, n, m, k, d, seed)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), wx.view(np.uint64)), ("newton " + prec, n, m, k, d, seed)
    print(f"case {c}: n={n} m={m} k={k} d={d} B={B} ok (dd fast {e:.2e})", flush=True)
# ragged systems (per-polynomial m, per-term k): complex double and dd reference order bit-exact
# with the ragged restatement, dd fast order within the tolerance
for c in range(cases // 2):
    n = int(rng.integers(1, 40))
    d = int(rng.choice([1, 2, 3, 6]))
    mlo = int(rng.integers(1, 20)); mhi = mlo + int(rng.integers(0, 40))
    klo = int(rng.integers(1, min(n, 10) + 1)); khi = min(n, klo + int(rng.integers(0, 8)))
    B = int(rng.choice([1, 5, 64, 300]))
    seed = int(rng.integers(1, 1 << 30))
    r = pj.random_ragged_system(n, (mlo, mhi), (klo, khi), d, seed)
    ctx = pj.EvaluationContext(r)
    R = r.as_dict()
    pts = pj.random_points(n, B, seed + 3)
    p2 = np.stack([pts.real, pts.imag], -1)
    p4 = pj.to_dd(pts)
    got = ctx.evaluate_host(p2, "d")
    want = O.evaluate_ragged("d", R, p2)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), ("ragged d", n, d, mlo, mhi, klo, khi, seed)
    want4, ms = O.evaluate_ragged("dd", R, p4, magsum=True)
    assert np.array_equal(ctx.evaluate_dd(p4, order="ref").view(np.uint64), want4.view(np.uint64)), ("ragged dd ref", seed)
    e = dd_rel(ctx.evaluate_dd(p4), want4, ms)
    assert e <= 1e-30, ("ragged dd fast", seed, e)
    print(f"ragged {c}: n={n} d={d} m=[{mlo},{mhi}] k=[{klo},{khi}] B={B} ok", flush=True)
# the wide encoding (n > 256)
for c in range(4):
    n = int(rng.integers(257, 700))
    s = pj.random_system(n, int(rng.integers(1, 4)), int(rng.integers(1, 6)), int(rng.choice([2, 4])), 11 + c)
    ctx = pj.EvaluationContext(s, wide=True)
    S = sysd(s)
    pts = pj.random_points(n, 2, 5 + c)
    p2 = np.stack([pts.real, pts.imag], -1)
    got = ctx.evaluate_host(p2, "d")
    assert np.array_equal(got.view(np.uint64), O.evaluate("d", S, p2).view(np.uint64)), ("wide d", n)
    p4 = pj.to_dd(pts)
    want4, ms = O.evaluate("dd", S, p4, magsum=True)
    assert np.array_equal(ctx.evaluate_dd(p4, order="ref").view(np.uint64), want4.view(np.uint64)), ("wide ref", n)
    assert dd_rel(ctx.evaluate_dd(p4), want4, ms) <= 1e-30, ("wide fast", n)
    print(f"wide {c}: n={n} ok", flush=True)
print(f"all {cases} uniform, {cases // 2} ragged and 4 wide cases ok; worst uniform dd fast error {worst:.3e} x sum|terms|")

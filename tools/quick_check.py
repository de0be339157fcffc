"""Developer smoke: parity of every kernel variant against the oracle on C1/C3-shaped
systems plus a rough device timing. Not part of the test suite (see tests/)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1201_0499_b200 as pj
from oracle import oracle as O


def sysd(s):
    return dict(n=s.n, m=s.m, k=s.k, d=s.d, pos=s.positions.reshape(-1).copy(), exps=s.exponents.reshape(-1).copy(),
                coeffs=s.coeffs.copy())


for (n, m, k, d, B) in [(32, 32, 8, 2, 256), (64, 64, 16, 10, 16), (8, 3, 3, 5, 64), (4, 4, 1, 1, 64), (40, 40, 20, 3, 8),
                         (6, 4, 2, 3, 64)]:
    s = pj.random_system(n, m, k, d, 7)
    S = sysd(s)
    ctx = pj.EvaluationContext(s)
    pts = pj.random_points(n, B, 11)
    p2 = np.stack([pts.real, pts.imag], -1)
    t0 = time.time()
    got_d = ctx.evaluate_host(p2, "d")
    want_d = O.ref_evaluate(S, p2) if O.ref_available() else O.evaluate("d", S, p2)
    ok_d = np.array_equal(got_d.view(np.uint64), want_d.view(np.uint64))
    p4 = pj.to_dd(pts)
    p4[..., 1] = p4[..., 0] * 2.0 ** -60 * 0.37
    p4[..., 3] = p4[..., 2] * 2.0 ** -61 * -0.73
    want_dd, ms = O.evaluate("dd", S, p4, magsum=True)
    got_ref = ctx.evaluate_dd(p4, order="ref")
    ok_ref = np.array_equal(got_ref, want_dd)
    got_fast = ctx.evaluate_dd(p4)
    err = np.abs((got_fast[..., 0] - want_dd[..., 0]) + (got_fast[..., 1] - want_dd[..., 1]))
    err = np.maximum(err, np.abs((got_fast[..., 2] - want_dd[..., 2]) + (got_fast[..., 3] - want_dd[..., 3])))
    rel = np.max(err / np.maximum(ms, 1e-300))
    print(f"n={n} m={m} k={k} d={d}: d bit-exact={ok_d} dd-ref==oracle={ok_ref} dd-fast max|err|/sum|terms|={rel:.3e}"
          f" launch={ctx.launch('dd')}", flush=True)

# timing C1 65536 points
s = pj.random_system(32, 32, 8, 2, 7)
ctx = pj.EvaluationContext(s)
B = 65536
pts = torch.from_numpy(pj.to_dd(pj.random_points(32, B, 11))).cuda()
out = torch.empty((B, 32 + 1024, 4), dtype=torch.float64, device="cuda")
for prec, W in (("dd", 4), ("d", 2)):
    pin = pts if W == 4 else pts[..., [0, 2]].contiguous()
    o = out if W == 4 else torch.empty((B, 1056, 2), dtype=torch.float64, device="cuda")
    for _ in range(3):
        ctx.evaluate_device(pin, o, prec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ctx.evaluate_device(pin, o, prec)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    flops = 3891200 if prec == "dd" else 282624
    print(f"{prec}: {ms:.3f} ms / {B} pts -> {B / ms * 1e3:.3e} evals/s, model {B * flops / ms / 1e9:.2f} TFLOP/s",
          ctx.launch(prec))
print("fp64 peak probe TF:", pj.fp64_peak_tflops())

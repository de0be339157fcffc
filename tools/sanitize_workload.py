"""Small workload touching every kernel through the host API (no torch kernels), for
compute-sanitizer memcheck / racecheck / synccheck / initcheck runs (tools/sanitize.sh)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1201_0499_b200 as pj


def pts(n, B, seed, prec):
    z = pj.random_points(n, B, seed)
    if prec == "d":
        return np.stack([z.real, z.imag], -1)
    p = pj.to_dd(z)
    p[..., 1] = p[..., 0] * 2.0 ** -55
    return p


cases = [
    ((32, 32, 8, 2), False, 5),    # fast dd, fast d, generic dd-ref
    ((8, 3, 3, 5), False, 7),      # d > 2 power tables
    ((24, 20, 16, 3), False, 3),   # k = 16
    ((40, 40, 20, 3), False, 2),   # k > 16: generic kernel in both orders
    ((10, 70, 4, 3), False, 3),    # m > 32: chunks and accumulators
    ((300, 2, 3, 3), True, 2),     # wide encoding
    ((200, 2, 3, 255), False, 1),  # global-scratch tables
]
for (n, m, k, d), wide, B in cases:
    s = pj.random_system(n, m, k, d, 7)
    ctx = pj.EvaluationContext(s, wide=wide)
    ctx.evaluate_host(pts(n, B, 11, "d"), "d")
    ctx.evaluate_dd(pts(n, B, 11, "dd"))
    ctx.evaluate_dd(pts(n, B, 11, "dd"), order="ref")
    if n <= 256:
        ctx.newton_host(pts(n, B, 11, "dd"), "dd", iters=2)
        ctx.newton_host(pts(n, B, 11, "d"), "d", iters=1)
    if n <= 32:
        ctx.newton_host(pts(n, B, 11, "dd"), "mixed", iters=2)
    print(f"ok n={n} m={m} k={k} d={d}", flush=True)
# Newton with a global slab (n > 64 dd) and the pipelined host path with several chunks
s = pj.random_system(100, 7, 5, 4, 7)
pj.EvaluationContext(s).newton_host(pts(100, 3, 5, "dd"), "dd")
print("ok", flush=True)

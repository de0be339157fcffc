"""Sweep fast-kernel variants and launch shapes on a B200; print evals/s and the model
FP64 fraction. Also checks every variant against the oracle (dd, tolerance contract).

    python tools/tune.py [--quick]
"""
import itertools
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1201_0499_b200 as pj
from oracle import oracle as O

def model_flops(n, m, k, d):
    return (n * max(d - 2, 0) + n * m * (k - 1) + n * m * (5 * k - 4)) * 80 + n * m * (k + 1) * 40


def timeit(ctx, pts, out, reps=5):
    for _ in range(2):
        ctx.evaluate_device(pts, out, "dd")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ctx.evaluate_device(pts, out, "dd")
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    quick = "--quick" in sys.argv
    peak = pj.fp64_peak_tflops()
    print(f"fp64 peak {peak:.2f} TF", flush=True)
    cases = [(32, 32, 8, 2, 65536), (64, 64, 16, 10, 16384)]
    for (n, m, k, d, B) in cases:
        s = pj.random_system(n, m, k, d, 7)
        S = dict(n=n, m=m, k=k, d=d, pos=s.positions.reshape(-1).copy(), exps=s.exponents.reshape(-1).copy(),
                 coeffs=s.coeffs.copy())
        ctx = pj.EvaluationContext(s)
        p4 = pj.to_dd(pj.random_points(n, B, 11))
        pts = torch.from_numpy(p4).cuda()
        out = torch.empty((B, n + n * n, 4), dtype=torch.float64, device="cuda")
        want, ms = O.evaluate("dd", S, p4[:8], magsum=True, threads=8)
        variants = [1] if quick else [-1, 1]
        shapes = [(0, 0), (256, 1), (256, 2)] if quick else [(0, 0), (64, 1), (64, 2), (96, 2), (128, 1), (128, 2), (160, 2), (192, 2),
                                         (256, 1), (256, 2), (256, 4)]
        for v in variants:
            for (th, tp) in shapes:
                try:
                    ctx.set_variant(v)
                    ctx.set_launch("dd", th, tp)
                except Exception as exc:
                    print(f"  variant {v} th {th} tp {tp}: {exc}")
                    continue
                L = ctx.launch("dd")
                ms_ = timeit(ctx, pts, out)
                got = out[:8].cpu().numpy()
                e = np.maximum(np.abs((got[..., 0] - want[..., 0]) + (got[..., 1] - want[..., 1])),
                               np.abs((got[..., 2] - want[..., 2]) + (got[..., 3] - want[..., 3])))
                rel = float(np.max(e[ms > 0] / ms[ms > 0]))
                tf = model_flops(n, m, k, d) * B / (ms_ * 1e-3) / 1e12
                print(f"n={n} k={k} d={d} variant={v:3d} launch={L} {ms_:8.3f} ms {B / ms_ * 1e3:12.4e} evals/s "
                      f"model {tf:6.2f} TF frac {tf / peak:.3f} err {rel:.2e}", flush=True)
        ctx.set_variant(0)
        ctx.set_launch("dd", 0, 0)


if __name__ == "__main__":
    main()

"""Developer: Newton solve timing at C2 (n=32, 65,536 points) and C3 (n=64, 8,192) for the library
named by PJ_LIB_PATH (variant comparisons)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1201_0499_b200 as pj

tag = os.path.basename(os.environ.get("PJ_LIB_PATH", "default"))
cases = [(32, 32, 8, 2, 65536), (64, 64, 16, 10, 8192)][: int(os.environ.get("PJ_NCASES", "2"))]
for (n, m, k, d, B) in cases:
    s = pj.random_system(n, m, k, d, 7)
    ctx = pj.EvaluationContext(s)
    thr = int(os.environ.get("PJ_NT_THREADS", "0"))
    for prec in os.environ.get("PJ_PRECS", "dd,d").split(","):
        if prec == "mixed" and n > 32:
            continue
        if thr:
            ctx.set_launch(prec, thr, newton=True)
        W = 4 if prec in ("dd", "mixed") else 2
        pts = pj.random_points(n, B, 11)
        p = pj.to_dd(pts) if W == 4 else np.stack([pts.real, pts.imag], -1)
        x = torch.from_numpy(p).cuda()
        work = torch.empty((B, n + n * n, W), dtype=torch.float64, device="cuda")
        out = torch.empty_like(x)
        ctx.evaluate_device(x, work, "dd" if W == 4 else prec)
        for _ in range(2):
            ctx.newton_solve_device(work, x, out, prec)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            ctx.newton_solve_device(work, x, out, prec)
        e1.record()
        torch.cuda.synchronize()
        ts = e0.elapsed_time(e1) / 5
        print(f"{tag} n={n} {prec}: solve {ts:.3f} ms ({B / ts / 1e3:.3f} M/s) {ctx.launch(prec, newton=True)}", flush=True)

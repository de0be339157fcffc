"""One evaluation + one Newton solve of C2 (65,536 points, complex dd) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1201_0499_b200 as pj

n = int(os.environ.get("PJ_N", "32"))
B = int(os.environ.get("PJ_B", "65536"))
prec = os.environ.get("PJ_PREC", "dd")
s = pj.random_system(n, n, 8 if n == 32 else 16, 2 if n == 32 else 10, 7)
ctx = pj.EvaluationContext(s)
thr = int(os.environ.get("PJ_NT_THREADS", "0"))
if thr:
    ctx.set_launch(prec, thr, newton=True)
W = 4 if prec == "dd" else 2
pts = pj.random_points(n, B, 11)
p = pj.to_dd(pts) if prec == "dd" else __import__("numpy").stack([pts.real, pts.imag], -1)
x = torch.from_numpy(p).cuda()
work = torch.empty((B, n + n * n, W), dtype=torch.float64, device="cuda")
out = torch.empty_like(x)
for _ in range(2):
    ctx.evaluate_device(x, work, prec)
    ctx.newton_solve_device(work, x, out, prec)
torch.cuda.synchronize()
print("launch", ctx.launch(prec, newton=True))

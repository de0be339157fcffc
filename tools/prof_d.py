"""Developer: complex-double evaluation of C2 (65,536 points) for ncu captures of the d kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1201_0499_b200 as pj

n, m, k, d, B = (int(x) for x in sys.argv[1:6]) if len(sys.argv) > 5 else (32, 32, 8, 2, 65536)
th = int(os.environ.get("PJ_THREADS", "0"))
tp = int(os.environ.get("PJ_TP", "0"))
s = pj.random_system(n, m, k, d, 7)
ctx = pj.EvaluationContext(s)
if th or tp:
    ctx.set_launch("d", th, tp)
pts = pj.random_points(n, B, 11)
x = torch.from_numpy(np.stack([pts.real, pts.imag], -1)).cuda()
out = torch.empty((B, n + n * n, 2), dtype=torch.float64, device="cuda")
for _ in range(3):
    ctx.evaluate_device(x, out, "d")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    ctx.evaluate_device(x, out, "d")
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"d n={n}: {ms:.3f} ms, {B / ms / 1e3:.2f} M evals/s, launch {ctx.launch('d')}")

"""Developer: C3 (n = 64, k = 16, d = 10, 65,536 points, dd fast) at several CTA shapes
(pj_set_launch threads / tile points) — evals/s per shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1201_0499_b200 as pj

s = pj.random_system(64, 64, 16, 10, 7)
ctx = pj.EvaluationContext(s)
B = 65536
pts = [torch.from_numpy(pj.to_dd(pj.random_points(64, B, 11 + i))).cuda() for i in range(2)]
out = torch.empty((B, 64 + 64 * 64, 4), dtype=torch.float64, device="cuda")
shapes = [tuple(map(int, x.split("x"))) for x in os.environ.get("PJ_SHAPES", "0x0,256x2,256x1,288x1,320x1,352x1,320x2").split(",")]
for thr, tp in shapes:
    try:
        if thr:
            ctx.set_launch("dd", thr, tp)
    except Exception as e:  # noqa: BLE001
        print(thr, tp, "refused:", e, flush=True)
        continue
    for i in range(2):
        ctx.evaluate_device(pts[i % 2], out, "dd")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(6):
        ctx.evaluate_device(pts[i % 2], out, "dd")
    e1.record()
    torch.cuda.synchronize()
    print(thr, tp, ctx.launch("dd"), f"{B * 6 / (e0.elapsed_time(e1) * 1e-3) / 1e6:.3f} M evals/s", flush=True)

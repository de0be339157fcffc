"""Developer: C2 (or C3 with C3=1) fast dd throughput per (threads, tile points) launch shape."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1201_0499_b200 as pj
import os
n, m, k, d, B = (64, 64, 16, 10, 8192) if os.environ.get("C3") else (32, 32, 8, 2, 65536)
s = pj.random_system(n, m, k, d, 7)
ctx = pj.EvaluationContext(s)
pts = [torch.from_numpy(pj.to_dd(pj.random_points(n, B, 11 + i))).cuda() for i in range(2)]
out = torch.empty((B, n + n * n, 4), dtype=torch.float64, device="cuda")
for th, tp in ([(256, 2), (320, 1), (320, 2), (384, 1), (352, 1), (256, 1)] if os.environ.get("C3") else [(256, 2), (256, 3)]):
    try:
        ctx.set_launch("dd", th, tp)
    except Exception as e:
        print(th, tp, "refused", e); continue
    L = ctx.launch("dd")
    for i in range(3): ctx.evaluate_device(pts[i % 2], out, "dd")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20): ctx.evaluate_device(pts[i % 2], out, "dd")
    e1.record(); torch.cuda.synchronize()
    print(th, tp, L, f"{B * 20 / (e0.elapsed_time(e1) * 1e-3) / 1e6:.3f}M", flush=True)

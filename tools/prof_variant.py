"""One timed launch per requested fast-kernel variant at C1 (for ncu captures).
    python tools/prof_variant.py <variant> [threads tile] [n m k d B]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1201_0499_b200 as pj

v = int(sys.argv[1])
th = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tp = int(sys.argv[3]) if len(sys.argv) > 3 else 0
n, m, k, d, B = (int(x) for x in sys.argv[4:9]) if len(sys.argv) > 8 else (32, 32, 8, 2, 65536)
s = pj.random_system(n, m, k, d, 7)
ctx = pj.EvaluationContext(s)
ctx.set_variant(v)
ctx.set_launch("dd", th, tp)
print(ctx.launch("dd"))
pts = torch.from_numpy(pj.to_dd(pj.random_points(n, B, 11))).cuda()
out = torch.empty((B, n + n * n, 4), dtype=torch.float64, device="cuda")
for _ in range(3):
    ctx.evaluate_device(pts, out, "dd")
torch.cuda.synchronize()
